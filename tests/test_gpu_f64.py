"""GPU parity of the FP64-output option (include/stkde.h
stkde_compute_*_f64) against the FP64 oracle, through the C ABI.

The FP64 kernel evaluates every gate and every factor k_s, k_t with Alg. 1's IEEE
operation sequence, so they equal the oracle's doubles; it sums
acc = fma(k_s, k_t, acc) in another order.  With m <= n non-negative terms per voxel
the oracle's sum is within (m + 1) u f of the exact one (u = 2^-53: product and sum
roundings; adaptive: + one for the division by hs_i^2 ht_i), the kernel's within
(m + 1) u f (one rounding per fma, + one for k_s / (hs_i^2 ht_i)), and each final
division adds u/2: the test uses rtol = 2 (n + 2) u per voxel (rigorous), and the
support mask (f > 0) must agree EXACTLY at every voxel -- no ambiguity list is needed
because the gates are bitwise the oracle's.
"""
import os

import numpy as np
import pytest

import stkde_synth as synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

U = 2.0 ** -53


@pytest.fixture(scope="module")
def S():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1705_09366_b200 as S
    S.load_library()
    return S


def G(Gx, Gy, Gt, res=1.0, hs=3.0, ht=2.0, origin=(0.0, 0.0, 0.0), tres=None):
    return dict(x0=origin[0], y0=origin[1], t0=origin[2], sres=res, tres=res if tres is None else tres,
                Gx=Gx, Gy=Gy, Gt=Gt, hs=hs, ht=ht)


def make_points(n, g, clustered, seed):
    ext = (g["Gx"] * g["sres"], g["Gy"] * g["sres"], g["Gt"] * g["tres"])
    if clustered:
        p = synth.clustered_points(n, 4, 3 * g["sres"], 3 * g["tres"], ext, seed)
    else:
        p = synth.uniform_points(n, ext, seed)
    p = p + np.array([g["x0"], g["y0"], g["t0"]], np.float32)
    extra = np.array([[g["x0"] - 0.8 * g["hs"], g["y0"] + ext[1] / 2, g["t0"] + ext[2] / 2],
                      [g["x0"] + ext[0] + 0.5 * g["hs"], g["y0"] - 0.3 * g["hs"], g["t0"] - 0.5 * g["ht"]]],
                     np.float32)
    return np.concatenate([p, extra]).astype(np.float32)


def assert_f64_parity(gpu, ref, n, what=""):
    gpu = np.asarray(gpu, np.float64).reshape(-1)
    ref = np.asarray(ref, np.float64).reshape(-1)
    assert gpu.shape == ref.shape
    assert np.array_equal(gpu > 0, ref > 0), "%s: support mask differs at %d voxels" % (
        what, int(np.count_nonzero((gpu > 0) != (ref > 0))))
    assert np.all(gpu >= 0)
    rtol = 2 * (max(n, 1) + 2) * U
    err = np.abs(gpu - ref)
    bad = err > rtol * np.abs(ref)
    assert not bad.any(), "%s: %d voxels beyond rtol %.2e (worst rel %.3e)" % (
        what, int(bad.sum()), rtol, float((err / np.maximum(np.abs(ref), 1e-300)).max()))
    nz = ref > 0
    return float((err[nz] / ref[nz]).max()) if nz.any() else 0.0


def run_f64(S, pts, kernel=0, t_begin=0, t_end=None, bw=None, **g):
    dev = torch.device("cuda", 0)
    with S.Plan(max_n=max(len(pts), 1), kernel=kernel, device=0, **g) as p:
        t = torch.from_numpy(np.ascontiguousarray(pts, np.float32)).to(dev)
        b = None if bw is None else torch.from_numpy(bw).to(dev)
        out = p.compute_f64(t, t_begin=t_begin, t_end=t_end, bw=b)
        torch.cuda.synchronize()
        p.check()
        return out.cpu().numpy()


@pytest.fixture(params=[2, 1, 0], ids=["tc", "mma", "simt"])
def engine(request):
    old = os.environ.get("STKDE_ENGINE")
    os.environ["STKDE_ENGINE"] = str(request.param)
    yield request.param
    if old is None:
        del os.environ["STKDE_ENGINE"]
    else:
        os.environ["STKDE_ENGINE"] = old


CASES = [
    # name, n, grid, kernel, clustered
    ("ragged", 500, G(37, 29, 41, hs=3.0, ht=2.0), 0, True),
    ("ragged_deep", 800, G(45, 33, 70, hs=5.5, ht=7.0), 0, True),
    ("classical", 600, G(33, 47, 35, hs=4.0, ht=3.0), 1, True),
    ("world_units", 700, G(50, 40, 30, res=0.37, hs=1.5, ht=1.2, origin=(1000.5, -2000.25, 30.0), tres=0.41), 0, True),
    ("big_disc", 200, G(80, 70, 40, hs=30.0, ht=6.0), 0, False),
    ("deep_window", 400, G(40, 36, 90, hs=5.0, ht=18.0), 0, True),   # H_t >= 16: 32-layer blocks
    ("one_voxel_grid", 50, G(1, 1, 1, hs=2.0, ht=2.0), 0, False),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_f64_small_full_parity(S, oracle_mod, case, engine):
    name, n, g, kid, clustered = case
    pts = make_points(n, g, clustered, seed=len(name) + 3)
    gpu = run_f64(S, pts, kernel=kid, **g)
    ref = oracle_mod.stkde_pb(pts, kernel=kid, with_ambiguity=False, **g)
    rel = assert_f64_parity(gpu, ref.vol, len(pts), what=name)
    print("%s: max rel %.3e" % (name, rel))


@pytest.mark.parametrize("name", ["tiny", "dengue"])
def test_f64_config_full_parity(S, oracle_mod, name):
    w = synth.make_config(name)
    g = w.grid_kwargs()
    gpu = run_f64(S, w.points, **g)
    ref = oracle_mod.stkde_pb(w.points, with_ambiguity=False, **g)
    rel = assert_f64_parity(gpu, ref.vol, w.n, what=name)
    print("%s: max rel %.3e" % (name, rel))


@pytest.mark.parametrize("name", ["ornith", "stress"])
def test_f64_full_size_sampled(S, oracle_mod, name):
    # BASELINE.json's largest configs at full size (ornith: 16-layer blocks, stress: 32):
    # sampled voxels -- the densest, random support voxels, random voxels, chosen on the
    # device so the float64 grid never leaves it -- against Alg. 1 voxel by voxel.
    w = synth.make_config(name)
    g = w.grid_kwargs()
    dev = torch.device("cuda", 0)
    with S.Plan(max_n=w.n, device=0, **g) as p:
        pts = torch.from_numpy(w.points).to(dev)
        out = p.compute_f64(pts).reshape(-1)
        torch.cuda.synchronize()
        p.check()
        r = synth.SplitMix64(23)
        top = torch.topk(out, 300).indices
        cand = torch.from_numpy((r.uniform01(200000) * out.numel()).astype(np.int64) % out.numel()).to(dev)
        sup = cand[out[cand] > 0][:300]
        rnd = torch.from_numpy((r.uniform01(100) * out.numel()).astype(np.int64) % out.numel()).to(dev)
        vox = torch.unique(torch.cat([top, sup, rnd]))
        gv = out[vox].cpu().numpy()
        vox = vox.cpu().numpy()
        del out
    val, _, _ = oracle_mod.stkde_vb_voxels(w.points, vox, **g)
    assert (val > 0).sum() >= 300
    rel = assert_f64_parity(gv, val, w.n, what=name)
    print("%s sampled: max rel %.3e over %d voxels" % (name, rel, len(vox)))


@pytest.mark.parametrize("ht", [9.0, 20.0], ids=["tl16", "tl32"])
def test_f64_slabs_bitwise_and_deterministic(S, oracle_mod, ht):
    g = G(40, 36, 150, hs=6.0, ht=ht)
    pts = make_points(700, g, True, seed=41)
    full = run_f64(S, pts, **g)
    again = run_f64(S, pts, **g)
    assert np.array_equal(full.view(np.uint64), again.view(np.uint64))
    for t0, t1 in [(0, 150), (5, 37), (37, 38), (64, 150), (149, 150)]:
        sl = run_f64(S, pts, t_begin=t0, t_end=t1, **g)
        assert np.array_equal(sl.view(np.uint64), full[:, :, t0:t1].view(np.uint64)), (t0, t1)
    ref = oracle_mod.stkde_pb(pts, with_ambiguity=False, **g)
    assert_f64_parity(full, ref.vol, len(pts), what="slab case")


def test_f64_matches_fp32_path(S):
    # the FP32 product path is within its north_star tolerance of the FP64 option
    w = synth.make_config("dengue")
    g = w.grid_kwargs()
    dev = torch.device("cuda", 0)
    with S.Plan(max_n=w.n, device=0, **g) as p:
        t = torch.from_numpy(w.points).to(dev)
        f32 = p.compute(t).double()
        f64 = p.compute_f64(t)
        torch.cuda.synchronize()
    assert float((f32 - f64).abs().max()) <= 1e-5 * float(f64.max())


def test_f64_adaptive_parity(S, oracle_mod):
    g = G(45, 33, 41, hs=5.5, ht=3.0)
    pts = make_points(600, g, True, seed=77)
    r = synth.SplitMix64(78)
    v = r.uniform01(2 * len(pts)).reshape(-1, 2)
    bw = ((0.25 + 0.75 * v) * np.array([g["hs"], g["ht"]])).astype(np.float32)
    bw[:50] = np.array([5.5, 3.0], np.float32)
    gpu = run_f64(S, pts, bw=bw, **g)
    ref = oracle_mod.stkde_pb_adaptive(pts, bw, with_ambiguity=False, **g)
    rel = assert_f64_parity(gpu, ref.vol, len(pts), what="adaptive")
    print("adaptive: max rel %.3e" % rel)
    sl = run_f64(S, pts, bw=bw, t_begin=7, t_end=30, **g)
    assert np.array_equal(sl.view(np.uint64), gpu[:, :, 7:30].view(np.uint64))


def test_f64_adaptive_classical_world_units(S, oracle_mod):
    g = G(50, 40, 30, res=0.37, hs=1.5, ht=1.2, origin=(1000.5, -2000.25, 30.0), tres=0.41)
    pts = make_points(500, g, True, seed=91)
    r = synth.SplitMix64(92)
    v = r.uniform01(2 * len(pts)).reshape(-1, 2)
    cap = np.array([np.float32(1.5), np.nextafter(np.float32(1.2), np.float32(0))], np.float32)
    bw = np.minimum(((0.3 + 0.7 * v) * np.array([1.5, 1.2])).astype(np.float32), cap)
    gpu = run_f64(S, pts, kernel=1, bw=bw, **g)
    ref = oracle_mod.stkde_pb_adaptive(pts, bw, kernel=1, with_ambiguity=False, **g)
    assert_f64_parity(gpu, ref.vol, len(pts), what="adaptive classical world units")


def test_f64_edge_cases(S):
    g = G(20, 20, 20, hs=3.0, ht=2.0)
    dev = torch.device("cuda", 0)
    with S.Plan(max_n=10, device=0, **g) as p:
        out = torch.full((20, 20, 20), 7.0, dtype=torch.float64, device=dev)
        p.compute_f64(torch.empty((0, 3), dtype=torch.float32, device=dev), out=out)
        torch.cuda.synchronize()
        assert float(out.abs().max()) == 0.0
        with pytest.raises(ValueError):
            p.compute_f64(torch.zeros((1, 3), dtype=torch.float32, device=dev),
                          out=torch.empty((20, 20, 20), dtype=torch.float32, device=dev))
        with pytest.raises(S.StkdeError):
            p.compute_f64(torch.zeros((1, 3), dtype=torch.float32, device=dev), t_begin=5, t_end=5)
        bad = torch.tensor([[5.0, float("nan"), 5.0], [10.0, 10.0, 10.0]], dtype=torch.float32, device=dev)
        p.compute_f64(bad)
        with pytest.raises(S.StkdeError):
            p.check()
