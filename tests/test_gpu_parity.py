"""GPU (CUDA, sm_100a) path vs the FP64 oracle, through the C ABI.

Element-wise parity at sizes the oracle finishes in seconds (several tiles,
ragged tails), sampled parity + exact properties at BASELINE.json's full sizes
in the launch configuration bench.py times, and the edge cases of the method.
"""
import os

import numpy as np
import pytest

import stkde_synth as synth
from parity import assert_parity

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _cuda_or_skip():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture(scope="module")
def S():
    _cuda_or_skip()
    import paper_1705_09366_b200 as S
    S.load_library()
    return S


def run_gpu(S, pts, kernel=0, **g):
    dev = torch.device("cuda", 0)
    with S.Plan(max_n=max(len(pts), 1), kernel=kernel, device=0, **g) as p:
        t = torch.from_numpy(np.ascontiguousarray(pts, np.float32)).to(dev)
        out = p.compute(t)
        c = p.count_contributions(t)
        torch.cuda.synchronize()
        p.check()
        info = p.info()
        return out.cpu().numpy(), int(c.item()), info


def G(Gx, Gy, Gt, res=1.0, hs=3.0, ht=2.0, origin=(0.0, 0.0, 0.0), tres=None):
    return dict(x0=origin[0], y0=origin[1], t0=origin[2], sres=res, tres=res if tres is None else tres,
                Gx=Gx, Gy=Gy, Gt=Gt, hs=hs, ht=ht)


SMALL = [
    # name, n, grid, kernel, clustered
    ("ragged_bt16", 500, G(37, 29, 41, hs=3.0, ht=2.0), 0, True),
    ("ragged_bt32", 800, G(45, 33, 70, hs=5.5, ht=7.0), 0, True),
    ("ragged_bt64", 300, G(40, 36, 150, hs=9.0, ht=20.0), 0, False),
    ("classical", 600, G(33, 47, 35, hs=4.0, ht=3.0), 1, True),
    ("world_units", 700, G(50, 40, 30, res=0.37, hs=1.5, ht=1.2, origin=(1000.5, -2000.25, 30.0), tres=0.41), 0, True),
    ("big_disc", 200, G(80, 70, 40, hs=30.0, ht=6.0), 0, False),
    ("one_voxel_grid", 50, G(1, 1, 1, hs=2.0, ht=2.0), 0, False),
    ("thin_slab", 400, G(64, 64, 3, hs=4.0, ht=1.0), 0, True),
    # bandwidths below one voxel: the disc / window holds at most the nearest voxel centre
    ("sub_voxel_bandwidth", 3000, G(40, 30, 20, hs=0.3, ht=0.4), 0, True),
    # classical kernel on Bt = 128 tiles (Gt > 64): small disc (H_s < 16, the PF = 1
    # loader instantiation) and large disc (H_s >= 16)
    ("classical_bt128_small", 900, G(45, 37, 150, hs=5.0, ht=6.0), 1, True),
    ("classical_bt128_large", 250, G(70, 60, 140, hs=18.0, ht=9.0), 1, False),
]


def make_points(n, g, clustered, seed):
    ext = (g["Gx"] * g["sres"], g["Gy"] * g["sres"], g["Gt"] * g["tres"])
    if clustered:
        p = synth.clustered_points(n, 4, 3 * g["sres"], 3 * g["tres"], ext, seed)
    else:
        p = synth.uniform_points(n, ext, seed)
    p = p + np.array([g["x0"], g["y0"], g["t0"]], np.float32)
    # points outside the box whose cylinders reach in (reading R6)
    extra = np.array([[g["x0"] - 0.8 * g["hs"], g["y0"] + ext[1] / 2, g["t0"] + ext[2] / 2],
                      [g["x0"] + ext[0] + 0.5 * g["hs"], g["y0"] - 0.3 * g["hs"], g["t0"] - 0.5 * g["ht"]]],
                     np.float32)
    return np.concatenate([p, extra]).astype(np.float32)


@pytest.fixture(params=[2, 1, 0, 3], ids=["tc", "mma", "simt", "ws"])
def engine(request):
    old = os.environ.get("STKDE_ENGINE")
    os.environ["STKDE_ENGINE"] = str(request.param)
    yield request.param
    if old is None:
        del os.environ["STKDE_ENGINE"]
    else:
        os.environ["STKDE_ENGINE"] = old


@pytest.mark.parametrize("case", SMALL, ids=[c[0] for c in SMALL])
def test_small_full_parity(S, oracle_mod, case, engine, monkeypatch):
    name, n, g, kid, clustered = case
    if "bt128" in name and engine == 2:   # small grids default to Bt = 64 (< 8 Bt-128 tiles per SM)
        monkeypatch.setenv("STKDE_BT", "128")
    pts = make_points(n, g, clustered, seed=len(name))
    gpu, C, info = run_gpu(S, pts, kernel=kid, **g)
    # the short-window engine takes H_t <= 8 (and H_s <= 120); other plans fall back to tcgen05
    ht_vox = int(np.ceil(g["ht"] / g["tres"]))
    assert info["engine"] == (2 if engine == 3 and ht_vox > 8 else engine)
    ref = oracle_mod.stkde_pb(pts, kernel=kid, **g)
    assert_parity(gpu, ref.vol, ref.slack, ref.amb, what=name)
    assert C == ref.contributions


@pytest.mark.parametrize("name", ["tiny", "dengue", "social"])
def test_config_full_parity(S, oracle_mod, name, engine):
    w = synth.make_config(name)
    g = w.grid_kwargs()
    gpu, C, info = run_gpu(S, w.points, **g)
    ref = oracle_mod.stkde_pb(w.points, **g)
    rel = assert_parity(gpu, ref.vol, ref.slack, ref.amb, what=name)
    assert C == ref.contributions
    print("%s: max |gpu-oracle|/max = %.3e, C = %d, tile %s" % (name, rel, C, (info["Bx"], info["By"], info["Bt"])))


def test_determinism_and_slabs(S, engine):
    w = synth.make_config("dengue")
    g = w.grid_kwargs()
    dev = torch.device("cuda", 0)
    t = torch.from_numpy(w.points).to(dev)
    with S.Plan(max_n=w.n, device=0, **g) as p:
        a = p.compute(t).clone()
        b = p.compute(t).clone()
        bt = p.info()["Bt"]
        assert torch.equal(a, b)
        # Bt-aligned and unaligned slabs equal the corresponding layers bitwise
        Gt = g["Gt"]
        for t0, t1 in [(0, min(bt, Gt)), (min(bt, Gt - 1), min(3 * bt, Gt)), (3, 50), (50, 51), (Gt - 5, Gt)]:
            s = p.compute_slab(t, t0, t1, n_norm=w.n)
            assert torch.equal(s, a[:, :, t0:t1]), (t0, t1)
        nparts = min(4, (Gt + bt - 1) // bt)       # at most one part per Bt block
        cuts = p.slab_partition(t, nparts)
        assert cuts[0] == 0 and cuts[-1] == g["Gt"] and all(c % bt == 0 for c in cuts[:-1])
        assert all(cuts[i] < cuts[i + 1] for i in range(nparts))


def test_split_hot_tiles(S, oracle_mod, engine):
    # Force tiny candidate chunks so most tiles split: the last-arriving chunk
    # sums the partials in chunk order (deterministic, parity-green).
    w = synth.make_config("dengue")
    g = w.grid_kwargs()
    os.environ["STKDE_CHUNK"] = "64"
    try:
        gpu, _, info = run_gpu(S, w.points, **g)
        gpu2, _, _ = run_gpu(S, w.points, **g)
    finally:
        del os.environ["STKDE_CHUNK"]
    # the slot budget may raise the chunk a little above the request; it stays
    # far below the hot tiles' candidate counts, so most of them split
    assert info["chunk_candidates"] <= 256
    assert np.array_equal(gpu, gpu2)
    ref = oracle_mod.stkde_pb(w.points, **g)
    assert_parity(gpu, ref.vol, ref.slack, ref.amb, what="split")


@pytest.mark.parametrize("bt_c", [(16, 4), (16, 8), (32, 8), (32, 16), (64, 16)])
def test_tile_variants(S, oracle_mod, bt_c):
    w = synth.make_config("tiny")
    g = w.grid_kwargs()
    os.environ["STKDE_BT"], os.environ["STKDE_CT"], os.environ["STKDE_ENGINE"] = str(bt_c[0]), str(bt_c[1]), "0"
    try:
        gpu, _, info = run_gpu(S, w.points, **g)
    finally:
        del os.environ["STKDE_BT"], os.environ["STKDE_CT"], os.environ["STKDE_ENGINE"]
    assert info["Bt"] == bt_c[0]
    ref = oracle_mod.stkde_pb(w.points, **g)
    assert_parity(gpu, ref.vol, ref.slack, ref.amb, what=str(bt_c))


@pytest.mark.parametrize("bt,bth", [(64, 16), (128, 16), (128, 8), (128, 64), (64, 128)])
def test_tc_tile_heights(S, oracle_mod, bt, bth):
    # tcgen05 engine at both tile heights and several home-bucket depths in T
    # (the candidate segments of a tile are the home blocks its reach meets)
    w = synth.make_config("dengue")
    g = w.grid_kwargs()
    os.environ["STKDE_BT"], os.environ["STKDE_BTH"], os.environ["STKDE_ENGINE"] = str(bt), str(bth), "2"
    try:
        gpu, _, info = run_gpu(S, w.points, **g)
    finally:
        del os.environ["STKDE_BT"], os.environ["STKDE_BTH"], os.environ["STKDE_ENGINE"]
    assert info["Bt"] == bt and info["By"] == 8 and info["engine"] == 2
    ref = oracle_mod.stkde_pb(w.points, **g)
    assert_parity(gpu, ref.vol, ref.slack, ref.amb, what="tc bt=%d bth=%d" % (bt, bth))


def test_sharded_single_process_equals_full(S):
    # stkde_compute_sharded with every "device" mapped to GPU 0 (fake multi-GPU):
    # slabs + the peer-memory gather kernel reproduce the full grid bitwise.
    w = synth.make_config("dengue")
    g = w.grid_kwargs()
    dev = torch.device("cuda", 0)
    t = torch.from_numpy(w.points).to(dev)
    plans = [S.Plan(max_n=w.n, device=0, **g) for _ in range(3)]
    try:
        full_ref = plans[0].compute(t).clone()
        cuts = plans[0].slab_partition(t, 3)
        slabs = [torch.empty((g["Gx"], g["Gy"], cuts[i + 1] - cuts[i]), device=dev) for i in range(3)]
        full = torch.full_like(full_ref, -1.0)
        used = S.compute_sharded(plans, [t] * 3, slabs, cuts=cuts, root=0, full=full)
        torch.cuda.synchronize()
        assert used == cuts
        assert torch.equal(full, full_ref)
    finally:
        for p in plans:
            p.close()


def test_edge_cases(S, oracle_mod):
    dev = torch.device("cuda", 0)
    g = G(20, 20, 20, hs=3.0, ht=2.0)
    # n = 0: zeros, no division
    with S.Plan(max_n=10, device=0, **g) as p:
        out = torch.full((20, 20, 20), 7.0, device=dev)
        p.compute(torch.zeros((0, 3), device=dev), out=out)
        assert not out.any()
        # n > max_n -> capacity error
        with pytest.raises(S.StkdeError) as e:
            p.compute(torch.zeros((11, 3), device=dev))
        assert e.value.code == -4
    # single point at a voxel centre: (3 pi / 8) / (hs^2 ht)
    pts = np.array([[10.5, 10.5, 10.5]], np.float32)
    gpu, C, _ = run_gpu(S, pts, **g)
    assert abs(gpu[10, 10, 10] / (3 * np.pi / 8 / (9 * 2)) - 1) < 1e-6
    ref = oracle_mod.stkde_pb(pts, **g)
    assert_parity(gpu, ref.vol, ref.slack, ref.amb, what="n=1")
    # non-finite coordinates are skipped and flagged
    bad = np.array([[5.0, 5.0, 5.0], [np.nan, 1.0, 1.0], [3.0, np.inf, 2.0]], np.float32)
    with S.Plan(max_n=3, device=0, **g) as p:
        out = p.compute(torch.from_numpy(bad).to(dev))
        with pytest.raises(S.StkdeError) as e:
            p.check()
        assert e.value.code == -5
        ref = oracle_mod.stkde_pb(bad, **g)
        assert_parity(out.cpu().numpy(), ref.vol, ref.slack, ref.amb, what="nonfinite")
    # invalid plans
    for bad_g in (dict(g, sres=0.0), dict(g, hs=-1.0), dict(g, Gt=0)):
        with pytest.raises(S.StkdeError) as e:
            S.Plan(max_n=1, device=0, **bad_g)
        assert e.value.code == -1


def test_tc_tma_store_edges(S, oracle_mod, monkeypatch):
    # tcgen05 engine, T-aligned output rows (Gt % 4 == 0 -> TMA tensor-store epilogue) on a
    # grid ragged in x, y and in the last T tile: the hardware-clipped box edges must match
    # the oracle; a 4-aligned slab (TMA path) and an unaligned one (fallback stores) must
    # equal the full grid's layers bitwise
    g = G(37, 29, 132, hs=5.0, ht=9.0)
    monkeypatch.setenv("STKDE_BT", "128")
    pts = make_points(700, g, True, seed=31)
    gpu, C, info = run_gpu(S, pts, **g)
    assert info["engine"] == 2 and info["Bt"] == 128
    ref = oracle_mod.stkde_pb(pts, **g)
    assert_parity(gpu, ref.vol, ref.slack, ref.amb, what="tma-edges")
    assert C == ref.contributions
    dev = torch.device("cuda", 0)
    with S.Plan(max_n=len(pts), device=0, **g) as p:
        t = torch.from_numpy(pts).to(dev)
        full = p.compute(t).cpu().numpy()
        for t0, t1 in ((4, 68), (3, 67), (64, 128), (32, 100), (96, 132), (128, 132), (0, 132)):
            s = p.compute_slab(t, t0, t1).cpu().numpy()
            assert np.array_equal(s, full[:, :, t0:t1]), (t0, t1)
        p.check()


def test_large_bandwidth_falls_back(S, oracle_mod):
    # H_s > 120 exceeds the tcgen05 engine's int8 chord table: the plan falls back to the
    # mma.sync engine, same parity contract
    g = G(270, 260, 12, hs=125.0, ht=3.0)
    pts = make_points(25, g, False, seed=33)
    gpu, C, info = run_gpu(S, pts, **g)
    assert info["engine"] == 1
    ref = oracle_mod.stkde_pb(pts, **g)
    assert_parity(gpu, ref.vol, ref.slack, ref.amb, what="hs>120")
    assert C == ref.contributions


@pytest.mark.parametrize("hs", [120.0, 119.5], ids=["hs120", "hs119.5"])
def test_largest_tc_bandwidth(S, oracle_mod, hs):
    # H_s = 120, the largest the tcgen05 engine's int8 chord offsets hold (and a non-integer
    # radius just under it): the tcgen05 engine, parity with the oracle
    g = G(260, 250, 40, hs=hs, ht=4.0)
    pts = make_points(20, g, False, seed=int(hs))
    gpu, C, info = run_gpu(S, pts, **g)
    assert info["engine"] == 2
    ref = oracle_mod.stkde_pb(pts, **g)
    assert_parity(gpu, ref.vol, ref.slack, ref.amb, what="hs=%g" % hs)
    assert C == ref.contributions


def test_partition_finer_than_bt(S):
    # more parts than Bt blocks (tcgen05 engine): the cost-balanced cuts refine to 32-layer
    # multiples, no slab is empty, and every slab equals the full grid's layers bitwise
    w = synth.make_config("dengue")            # Gt = 128 -> Bt = 64: 2 blocks
    g = w.grid_kwargs()
    dev = torch.device("cuda", 0)
    with S.Plan(max_n=w.n, device=0, **g) as p:
        assert p.info()["engine"] == 2
        t = torch.from_numpy(w.points).to(dev)
        full = p.compute(t).cpu().numpy()
        cuts = p.slab_partition(t, 4)
        assert cuts[0] == 0 and cuts[-1] == w.G[2]
        assert all(b > a for a, b in zip(cuts[:-1], cuts[1:])), cuts
        assert all(c % 32 == 0 for c in cuts[:-1]), cuts
        for a, b in zip(cuts[:-1], cuts[1:]):
            s = p.compute_slab(t, a, b, n_norm=w.n).cpu().numpy()
            assert np.array_equal(s, full[:, :, a:b]), (a, b)
        p.check()


@pytest.mark.parametrize("name", ["dengue", "social"])
def test_xslabs_equal_full_grid(S, name):
    # x-slabs (multiples of 16 columns, tcgen05 engine) are the full grid's rows, bitwise;
    # the cost-balanced x partition covers the grid with non-empty slabs
    w = synth.make_config(name)
    g = w.grid_kwargs()
    dev = torch.device("cuda", 0)
    with S.Plan(max_n=w.n, device=0, **g) as p:
        t = torch.from_numpy(w.points).to(dev)
        full = p.compute(t).cpu().numpy()
        for n in (3, 8):
            cuts = p.xslab_partition(t, n)
            assert cuts[0] == 0 and cuts[-1] == w.G[0] and all(b > a for a, b in zip(cuts[:-1], cuts[1:]))
            for a, b in zip(cuts[:-1], cuts[1:]):
                s = p.compute_xslab(t, a, b, n_norm=w.n).cpu().numpy()
                assert np.array_equal(s, full[a:b]), (a, b)
        p.check()


@pytest.mark.parametrize("eng", [2, 3], ids=["tc", "ws"])
def test_xslab_ragged_grid(S, oracle_mod, eng, monkeypatch):
    # ragged x / y / unaligned G_t: the last x-slab ends at G_x, slabs still equal the full grid
    # (tcgen05 and short-window engines; the latter's grid also against the oracle)
    monkeypatch.setenv("STKDE_ENGINE", str(eng))
    g = G(45, 33, 70, hs=5.5, ht=7.0)
    pts = make_points(800, g, True, seed=41)
    dev = torch.device("cuda", 0)
    with S.Plan(max_n=len(pts), device=0, **g) as p:
        assert p.info()["engine"] == eng
        t = torch.from_numpy(pts).to(dev)
        full = p.compute(t).cpu().numpy()
        if eng == 3:
            ref = oracle_mod.stkde_pb(pts, **g)
            assert_parity(full, ref.vol, ref.slack, ref.amb, what="ws ragged")
        for a, b in ((0, 16), (16, 45), (32, 45), (0, 45)):
            s = p.compute_xslab(t, a, b).cpu().numpy()
            assert np.array_equal(s, full[a:b]), (a, b)
        with pytest.raises(S.StkdeError):
            p.compute_xslab(t, 8, 24)                  # not a multiple of 16


@pytest.mark.parametrize("axis", ["x", "t"])
def test_sharded_driver_axes(S, axis):
    # the per-rank driver (sharded.ShardedSTKDE) for 3 ranks run in turn on one GPU: the
    # assembled x- or time-slabs are the single-GPU grid, bitwise
    from paper_1705_09366_b200.sharded import ShardedSTKDE, assemble
    w = synth.make_config("dengue")
    g = w.grid_kwargs()
    t = torch.from_numpy(w.points).to(torch.device("cuda", 0))
    with S.Plan(max_n=w.n, device=0, **g) as p:
        full = p.compute(t).cpu()
    slabs, cuts = [], None
    for r in range(3):
        d = ShardedSTKDE(t, grid=g, rank=r, world=3, axis=axis)
        slabs.append(d.compute().cpu())
        cuts = d.cuts
        d.close()
    assert torch.equal(assemble(slabs, cuts, w.G, axis=axis), full)


def test_sharded_x_single_process_equals_full(S):
    # stkde_compute_sharded_x with every "device" mapped to GPU 0: x-slabs + the per-device
    # peer copies into the root's grid reproduce the full grid bitwise; cuts from the device
    w = synth.make_config("dengue")
    g = w.grid_kwargs()
    dev = torch.device("cuda", 0)
    t = torch.from_numpy(w.points).to(dev)
    plans = [S.Plan(max_n=w.n, device=0, **g) for _ in range(3)]
    try:
        full_ref = plans[0].compute(t).clone()
        cuts = plans[0].xslab_partition(t, 3)
        slabs = [torch.empty((cuts[i + 1] - cuts[i], g["Gy"], g["Gt"]), device=dev) for i in range(3)]
        full = torch.full_like(full_ref, -1.0)
        used = S.compute_sharded(plans, [t] * 3, slabs, root=0, full=full, axis="x")
        torch.cuda.synchronize()
        assert used == cuts
        assert torch.equal(full, full_ref)
        # the fused gather: no slab buffers, every device's kernel stores into the root's grid
        full2 = torch.full_like(full_ref, float("nan"))
        used2 = S.compute_sharded(plans, [t] * 3, None, cuts=cuts, root=0, full=full2, axis="x")
        torch.cuda.synchronize()
        assert used2 == cuts
        assert torch.equal(full2, full_ref)
    finally:
        for p in plans:
            p.close()


@pytest.mark.parametrize("case", [c for c in SMALL if c[0].startswith("classical_bt128")], ids=lambda c: c[0])
def test_classical_bt128_slabs(S, oracle_mod, case, monkeypatch):
    # the classical kernel on Bt = 128 tiles (both loader instantiations) through
    # the slab calls: every slab equals the full grid's layers bitwise, the full grid the oracle
    name, n, g, kid, clustered = case
    monkeypatch.setenv("STKDE_BT", "128")
    pts = make_points(n, g, clustered, seed=len(name))
    dev = torch.device("cuda", 0)
    with S.Plan(max_n=len(pts), kernel=kid, device=0, **g) as p:
        assert p.info()["Bt"] == 128
        t = torch.from_numpy(pts).to(dev)
        full = p.compute(t).cpu().numpy()
        for t0, t1 in ((0, 64), (32, 96), (5, 133), (128, g["Gt"]), (0, g["Gt"])):
            s = p.compute_slab(t, t0, t1, n_norm=len(pts)).cpu().numpy()
            assert np.array_equal(s, full[:, :, t0:t1]), (t0, t1)
        p.check()
    ref = oracle_mod.stkde_pb(pts, kernel=kid, **g)
    assert_parity(full, ref.vol, ref.slack, ref.amb, what=name)


@pytest.mark.parametrize("name", ["tiny", "dengue"])
def test_graph_capture_replays_compute(S, name):
    # the compute call is CUDA-graph capturable (include/stkde.h): a captured pass replays
    # bitwise equal to a direct call, reads the point buffer as it is at launch time (refilled
    # in place with another point set), and a captured slab equals the direct slab
    w = synth.make_config(name)
    g = w.grid_kwargs()
    dev = torch.device("cuda", 0)
    other = synth.uniform_points(w.n, (g["Gx"] * g["sres"], g["Gy"] * g["sres"], g["Gt"] * g["tres"]), 99)
    with S.Plan(max_n=w.n, device=0, **g) as p:
        t = torch.from_numpy(w.points).to(dev)
        direct = p.compute(t).clone()
        gr = p.graph(t)
        for _ in range(3):
            out = gr.launch()
        torch.cuda.synchronize()
        assert torch.equal(out, direct)
        t.copy_(torch.from_numpy(other).to(dev))          # refill in place: the graph reads it
        out = gr.launch().clone()
        direct2 = p.compute(t).clone()
        torch.cuda.synchronize()
        assert torch.equal(out, direct2) and not torch.equal(direct2, direct)
        t0, t1 = 3, g["Gt"] - 5
        gs = p.graph(t, t_begin=t0, t_end=t1, n_norm=w.n)
        s = gs.launch().clone()
        torch.cuda.synchronize()
        assert torch.equal(s, direct2[:, :, t0:t1])
        if p.info()["engine"] == 2:                         # x-slabs: tcgen05 engine
            gx = p.graph_xslab(t, 16, min(48, g["Gx"]), n_norm=w.n)
            sx = gx.launch().clone()
            torch.cuda.synchronize()
            assert torch.equal(sx, direct2[16:min(48, g["Gx"])])
            gx.close()
        gr.close()
        gs.close()
        p.check()
