"""GPU parity of the adaptive-bandwidth estimator and the multi-bandwidth sweep
 against the FP64 oracle, through the C ABI.

Adaptive (reading R15): f = 1/n sum_i k_s k_t / (hs_i^2 ht_i) with the
point's own gates; oracle.stkde_pb_adaptive is pinned in
tests/test_oracle_adaptive_pins.py.  Sweep: grid k of stkde_compute_sweep is the
fixed-bandwidth density at (hs_k, ht_k) (oracle.stkde_pb, pinned in
tests/test_oracle_pins.py).  Same acceptance as test_gpu_parity.py.
"""
import os
import zlib

import numpy as np
import pytest

import stkde_synth as synth
from parity import assert_parity, cylinder_voxels

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


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


def f32_le(h):
    c = np.float32(h)
    return c if float(c) <= h else np.nextafter(c, np.float32(0))


def make_case(n, g, seed, lo=0.25, clustered=True):
    ext = (g["Gx"] * g["sres"], g["Gy"] * g["sres"], g["Gt"] * g["tres"])
    if clustered:
        p = synth.clustered_points(n, 4, 3 * g["sres"], 3 * g["tres"], ext, seed)
    else:
        p = synth.uniform_points(n, ext, seed)
    p = (p + np.array([g["x0"], g["y0"], g["t0"]], np.float32)).astype(np.float32)
    r = synth.SplitMix64(seed + 7)
    v = r.uniform01(2 * len(p)).reshape(-1, 2)
    cap = np.array([f32_le(g["hs"]), f32_le(g["ht"])], np.float32)
    bw = ((lo + (1 - lo) * v) * np.array([g["hs"], g["ht"]])).astype(np.float32)
    bw[: len(p) // 8] = cap
    return p, np.minimum(bw, cap)


CASES = [
    # name, n, grid, kernel
    ("bt128_ragged", 500, G(37, 29, 141, hs=4.0, ht=6.0), 0),
    ("bt64_ragged", 600, G(45, 33, 41, hs=5.5, ht=3.0), 0),
    ("classical", 500, G(33, 47, 70, hs=4.0, ht=3.0), 1),
    ("world_units", 600, G(50, 40, 30, res=0.37, hs=1.5, ht=1.2, origin=(1000.5, -2000.25, 30.0), tres=0.41), 0),
    ("big_disc", 150, G(80, 70, 40, hs=30.0, ht=6.0), 0),
    ("tiny_h", 400, G(40, 40, 40, hs=1.0, ht=1.0), 0),
]


def run_adaptive(S, pts, bw, kernel=0, **g):
    dev = torch.device("cuda", 0)
    with S.Plan(max_n=max(len(pts), 1), kernel=kernel, device=0, **g) as p:
        t = torch.from_numpy(pts).to(dev)
        b = torch.from_numpy(bw).to(dev)
        out = p.compute_adaptive(t, b)
        c = p.count_contributions_adaptive(t, b)
        torch.cuda.synchronize()
        p.check()
        return out.cpu().numpy(), int(c.item()), p.info()


@pytest.mark.parametrize("name,n,g,kernel", CASES, ids=[c[0] for c in CASES])
def test_adaptive_parity(S, oracle_mod, name, n, g, kernel, monkeypatch):
    if "bt128" in name:        # small grids default to Bt = 64
        monkeypatch.setenv("STKDE_BT", "128")
    pts, bw = make_case(n, g, seed=zlib.crc32(name.encode()) % 1000)
    gpu, C, info = run_adaptive(S, pts, bw, kernel=kernel, **g)
    assert info["engine"] == 2
    assert info["Bt"] == (128 if "bt128" in name else 64)
    ref = oracle_mod.stkde_pb_adaptive(pts, bw, kernel=kernel, **g)
    assert ref.vol.max() > 0
    assert_parity(gpu, ref.vol, ref.slack, ref.amb, what=name)
    assert C == ref.contributions == oracle_mod.contributions_adaptive(pts, bw, kernel=kernel, **g)


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("case", [0, 1], ids=["bt128", "bt64"])
def test_adaptive_parity_seeds(S, oracle_mod, case, seed, monkeypatch):
    # weights W_i / W_max span 64x here: the unbiased fixed-point sum (ICOMP)
    # keeps the small-weight points inside the tolerance
    name, n, g, kernel = CASES[case]
    if "bt128" in name:        # small grids default to Bt = 64
        monkeypatch.setenv("STKDE_BT", "128")
    pts, bw = make_case(n, g, seed=seed)
    gpu, C, _ = run_adaptive(S, pts, bw, kernel=kernel, **g)
    ref = oracle_mod.stkde_pb_adaptive(pts, bw, kernel=kernel, **g)
    assert_parity(gpu, ref.vol, ref.slack, ref.amb, what="%s seed %d" % (name, seed))
    assert C == ref.contributions


def test_adaptive_uniform_equals_fixed(S, oracle_mod):
    g = G(48, 40, 100, hs=5.0, ht=4.0)
    pts, _ = make_case(800, g, seed=3)
    bw = np.tile(np.array([[5.0, 4.0]], np.float32), (len(pts), 1))
    gpu_a, _, _ = run_adaptive(S, pts, bw, **g)
    dev = torch.device("cuda", 0)
    with S.Plan(max_n=len(pts), device=0, **g) as p:
        gpu_f = p.compute(torch.from_numpy(pts).to(dev)).cpu().numpy()
    ref = oracle_mod.stkde_pb(pts, **g)
    assert_parity(gpu_a, ref.vol, ref.slack, ref.amb, what="uniform-adaptive")
    assert np.abs(gpu_a.astype(np.float64) - gpu_f).max() <= 1e-5 * ref.vol.max()


def test_adaptive_deterministic_and_slab(S):
    g = G(40, 32, 260, hs=4.0, ht=9.0)
    pts, bw = make_case(1500, g, seed=9)
    dev = torch.device("cuda", 0)
    with S.Plan(max_n=len(pts), device=0, **g) as p:
        t, b = torch.from_numpy(pts).to(dev), torch.from_numpy(bw).to(dev)
        a = p.compute_adaptive(t, b).cpu().numpy()
        a2 = p.compute_adaptive(t, b).cpu().numpy()
        Bt = p.info()["Bt"]
        s = p.compute_adaptive_slab(t, b, Bt, 2 * Bt, n_norm=len(pts)).cpu().numpy()
        p.check()
    assert np.array_equal(a, a2)
    assert np.array_equal(s, a[:, :, Bt:2 * Bt])


def test_adaptive_bad_bandwidth_flagged(S, oracle_mod):
    g = G(30, 30, 30, hs=3.0, ht=2.0)
    pts, bw = make_case(200, g, seed=4)
    bw_bad = bw.copy()
    bw_bad[5] = [3.5, 1.0]          # above the plan's hs: skipped, flagged
    dev = torch.device("cuda", 0)
    with S.Plan(max_n=len(pts), device=0, **g) as p:
        out = p.compute_adaptive(torch.from_numpy(pts).to(dev), torch.from_numpy(bw_bad).to(dev)).cpu().numpy()
        with pytest.raises(S.StkdeError) as e:
            p.check()
        assert e.value.code == S.STKDE_EBANDWIDTH
        p.check()                   # the flag is cleared by the read
    keep = np.ones(len(pts), bool)
    keep[5] = False
    # the remaining points, normalised by the n passed in
    ref = oracle_mod.stkde_pb_adaptive(pts[keep], bw[keep], **g)
    scale = keep.sum() / len(pts)
    assert_parity(out, ref.vol * scale, ref.slack * scale, ref.amb, what="skip-bad-bw")


@pytest.mark.parametrize("eng", ["1", "3"], ids=["mma", "ws"])
def test_adaptive_needs_tc_engine(S, eng):
    old = os.environ.get("STKDE_ENGINE")
    os.environ["STKDE_ENGINE"] = eng
    try:
        g = G(20, 20, 20)
        pts, bw = make_case(50, g, seed=1)
        dev = torch.device("cuda", 0)
        with S.Plan(max_n=len(pts), device=0, **g) as p:
            with pytest.raises(S.StkdeError):
                p.compute_adaptive(torch.from_numpy(pts).to(dev), torch.from_numpy(bw).to(dev))
    finally:
        if old is None:
            os.environ.pop("STKDE_ENGINE")
        else:
            os.environ["STKDE_ENGINE"] = old


def test_adaptive_empty(S):
    g = G(20, 20, 20)
    dev = torch.device("cuda", 0)
    with S.Plan(max_n=10, device=0, **g) as p:
        out = torch.full(p.G, 7.0, device=dev)
        p.compute_adaptive(torch.empty((0, 3), device=dev), torch.empty((0, 2), device=dev), out=out)
        assert float(out.abs().max()) == 0.0


# ------------------------------------------------------------- sweep ---
@pytest.fixture(params=[2, 1, 0], ids=["tc", "mma", "simt"])
def engine(request):
    old = os.environ.get("STKDE_ENGINE")
    os.environ["STKDE_ENGINE"] = str(request.param)
    yield request.param
    if old is None:
        os.environ.pop("STKDE_ENGINE")
    else:
        os.environ["STKDE_ENGINE"] = old


def test_sweep_parity(S, oracle_mod, engine):
    g = G(45, 37, 90, hs=7.0, ht=6.0)
    ext = (45.0, 37.0, 90.0)
    pts = synth.clustered_points(900, 5, 4.0, 4.0, ext, 17)
    bws = [(7.0, 6.0), (4.5, 3.2), (2.2, 1.5), (0.9, 0.6)]
    dev = torch.device("cuda", 0)
    with S.Plan(max_n=len(pts), device=0, **g) as p:
        outs = p.compute_sweep(torch.from_numpy(pts).to(dev), [b[0] for b in bws], [b[1] for b in bws])
        torch.cuda.synchronize()
        p.check()
        assert p.info()["engine"] == engine
    for (hs, ht), o in zip(bws, outs):
        ref = oracle_mod.stkde_pb(pts, **dict(g, hs=hs, ht=ht))
        assert_parity(o.cpu().numpy(), ref.vol, ref.slack, ref.amb, what="sweep hs=%g ht=%g" % (hs, ht))


def test_sweep_matches_own_plans(S):
    g = G(64, 48, 130, hs=6.0, ht=8.0)
    pts = synth.clustered_points(3000, 6, 5.0, 6.0, (64.0, 48.0, 130.0), 23)
    bws = [(6.0, 8.0), (3.0, 5.0), (1.5, 2.0)]
    dev = torch.device("cuda", 0)
    t = torch.from_numpy(pts).to(dev)
    with S.Plan(max_n=len(pts), device=0, **g) as p:
        outs = [o.cpu().numpy() for o in p.compute_sweep(t, [b[0] for b in bws], [b[1] for b in bws])]
    for (hs, ht), o in zip(bws, outs):
        with S.Plan(max_n=len(pts), device=0, **dict(g, hs=hs, ht=ht)) as q:
            ref = q.compute(t).cpu().numpy()
        # same gates, same fixed-point codes, exact integer sums rounded once per voxel:
        # the sweep's grid is the narrower plan's grid, bitwise (support included)
        assert np.array_equal(o > 0, ref > 0), ((o > 0) != (ref > 0)).sum()
        assert np.array_equal(o, ref), np.abs(o.astype(np.float64) - ref).max() / ref.max()


def test_sweep_rejects_wider_bandwidth(S):
    g = G(20, 20, 20, hs=3.0, ht=2.0)
    dev = torch.device("cuda", 0)
    pts = synth.uniform_points(50, (20.0, 20.0, 20.0), 2)
    with S.Plan(max_n=50, device=0, **g) as p:
        with pytest.raises(S.StkdeError):
            p.compute_sweep(torch.from_numpy(pts).to(dev), [3.5], [2.0])


# ------------------------------------------- full sizes (bench.py --variant) ---
def _sample_voxels(gpu, points, g, rng, k_top=600, npts=400):
    # the densest GPU voxels plus an oracle-side sample (random points' cylinders and
    # uniform voxels, chosen without looking at the GPU output: a dropped support voxel
    # is caught wherever it is sampled)
    flat = gpu.reshape(-1)
    top = np.argpartition(flat, -k_top)[-k_top:]
    return np.unique(np.concatenate([top, cylinder_voxels(points, g, rng, npts=npts)]))


@pytest.mark.parametrize("name", ["social", "stress"])
def test_adaptive_full_size_sampled(S, oracle_mod, name):
    # the bench's adaptive workload (stkde_synth.adaptive_bandwidths) at the
    # BASELINE.json size: sampled voxels against adaptive Alg. 1, exact C
    w = synth.make_config(name)
    g = w.grid_kwargs()
    bw = synth.adaptive_bandwidths(w)
    gpu, C, _ = run_adaptive(S, w.points, bw, **g)
    vox = _sample_voxels(gpu, w.points, g, synth.SplitMix64(13))
    val, slack, amb = oracle_mod.stkde_vb_voxels_adaptive(w.points, bw, vox, **g)
    assert_parity(gpu.reshape(-1)[vox], val, slack, amb, vmax=max(val.max(), 0.0), what=name + "/adaptive")
    assert C == oracle_mod.contributions_adaptive(w.points, bw, **g)


def test_sweep_full_size_sampled(S, oracle_mod):
    # the bench's sweep (stress, f = 1 .. 0.25) at full size, sampled per grid
    w = synth.make_config("stress")
    g = w.grid_kwargs()
    dev = torch.device("cuda", 0)
    fr = synth.SWEEP_FRACTIONS
    with S.Plan(max_n=w.n, device=0, **g) as p:
        outs = p.compute_sweep(torch.from_numpy(w.points).to(dev), [f * w.hs for f in fr], [f * w.ht for f in fr])
        torch.cuda.synchronize()
        p.check()
        grids = [o.cpu().numpy() for o in outs]
        del outs
    for k, (f, gpu) in enumerate(zip(fr, grids)):
        gk = dict(g, hs=f * w.hs, ht=f * w.ht)
        vox = _sample_voxels(gpu, w.points, gk, synth.SplitMix64(17 + k), k_top=300, npts=300)
        val, slack, amb = oracle_mod.stkde_vb_voxels(w.points, vox, **gk)
        assert_parity(gpu.reshape(-1)[vox], val, slack, amb, vmax=max(val.max(), 0.0), what="sweep f=%g" % f)


def test_adaptive_xslabs_equal_full(S):
    # adaptive x-slabs (multiples of 16 columns) are the full adaptive grid's rows, bitwise
    w = synth.make_config("dengue")
    g = w.grid_kwargs()
    bw = synth.adaptive_bandwidths(w)
    dev = torch.device("cuda", 0)
    with S.Plan(max_n=w.n, device=0, **g) as p:
        t, b = torch.from_numpy(w.points).to(dev), torch.from_numpy(bw).to(dev)
        full = p.compute_adaptive(t, b).cpu().numpy()
        cuts = p.xslab_partition(t, 4)
        for a, c in zip(cuts[:-1], cuts[1:]):
            s = p.compute_adaptive_xslab(t, b, a, c, n_norm=w.n).cpu().numpy()
            assert np.array_equal(s, full[a:c]), (a, c)
        p.check()
