"""Seeded random plans: GPU (tcgen05 engine, through the C ABI) vs the FP64 oracle, every voxel.

The hand-picked cases of test_gpu_parity.py fix the tile heights, disc sizes and alignments
somebody thought of; here the plan itself is drawn (grid extents with ragged x / y / t tails,
G_t aligned or not to the 16-B TMA store, bandwidths from below one voxel to several tiles,
non-unit resolutions, far-from-zero origins, both kernels, uniform / clustered / coincident
points, points outside the box) from a fixed seed, so that a combination of template
instantiation, loader path and epilogue nobody listed still meets the oracle.  Every case is
also cut into a random time slab and a random x-slab, which must be the full grid's voxels
bitwise, and run twice (determinism).  PAPER.md:120-133 (definition),
Alg. 3 PAPER.md:302-335.
"""
import os

import numpy as np
import pytest

import stkde_synth as synth
from parity import assert_parity

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

NCASES = int(os.environ.get("STKDE_FUZZ_CASES", "40"))   # a one-off wider hunt: STKDE_FUZZ_CASES=2000


def draw_case(k):
    """Plan + points of fuzz case k; only the seeded generator module draws numbers."""
    r = synth.SplitMix64(0x5EED0000 + k)
    u = r.uniform01(24)
    Gx = 1 + int(u[0] * 90)
    Gy = 1 + int(u[1] * 70)
    Gt = [1 + int(u[2] * 40), 4 * (1 + int(u[2] * 12)), 65 + int(u[2] * 120), 128, 1 + int(u[2] * 300)][int(u[3] * 5) % 5]
    sres = [1.0, 0.37, 2.5, 1e-2][int(u[4] * 4) % 4]
    tres = [1.0, 0.41, 3.0, sres][int(u[5] * 4) % 4]
    # bandwidth in voxels: below one voxel ... a few tiles wide
    hs_v = [0.3 + 0.6 * u[6], 1.0 + 3.0 * u[6], 4.0 + 8.0 * u[6], 12.0 + 30.0 * u[6], float(2 + int(u[6] * 9))][int(u[7] * 5) % 5]
    ht_v = [0.3 + 0.6 * u[8], 1.0 + 3.0 * u[8], 4.0 + 6.0 * u[8], 10.0 + 40.0 * u[8], float(1 + int(u[8] * 8))][int(u[9] * 5) % 5]
    origin = [(0.0, 0.0, 0.0), (1000.5, -2000.25, 30.0), (-7.125, 3.5, -100.0)][int(u[10] * 3) % 3]
    g = dict(x0=origin[0], y0=origin[1], t0=origin[2], sres=sres, tres=tres, Gx=Gx, Gy=Gy, Gt=Gt,
             hs=hs_v * sres, ht=ht_v * tres)
    kernel = (k + int(u[11] * 4) // 3) % 2
    # keep the oracle in seconds: bound the expected number of contributions
    cyl = (2 * hs_v + 1) ** 2 * (2 * ht_v + 1)
    n = int(min(1 + u[12] * 3000, max(1.0, 4e7 / cyl)))
    ext = (Gx * sres, Gy * sres, Gt * tres)
    mode = int(u[13] * 4) % 4
    seed = 9000 + k
    if mode == 0:
        p = synth.uniform_points(n, ext, seed)
    elif mode == 1:
        p = synth.clustered_points(n, 1 + int(u[14] * 5), (0.5 + 4 * u[15]) * sres, (0.5 + 4 * u[16]) * tres, ext, seed)
    elif mode == 2:   # pile-up: many coincident points plus a uniform background
        p = synth.uniform_points(n, ext, seed)
        p[: n // 2] = p[0]
    else:             # points on voxel centres and voxel faces (gate arguments at lattice values)
        p = synth.uniform_points(n, ext, seed)
        p = (np.floor(p / np.array([sres, sres, tres], np.float32) * 2) / 2 * np.array([sres, sres, tres], np.float32)).astype(np.float32)
    p = p + np.array(origin, np.float32)
    outside = np.array([[origin[0] - 0.7 * g["hs"], origin[1] + ext[1] / 2, origin[2] + ext[2] / 2],
                        [origin[0] + ext[0] + 0.4 * g["hs"], origin[1] - 0.2 * g["hs"], origin[2] - 0.5 * g["ht"]],
                        [origin[0] + ext[0] / 2, origin[1] + ext[1] / 2, origin[2] + ext[2] + 0.9 * g["ht"]],
                        [origin[0] - 3 * g["hs"], origin[1], origin[2]]], np.float32)   # the last reaches nothing
    pts = np.ascontiguousarray(np.concatenate([p, outside]), np.float32)
    cut = (u[17], u[18], u[19], u[20])
    return g, kernel, pts, cut


def pile_up(k):
    """Draw k holds n/2 coincident points (mode 2 of draw_case)."""
    return int(synth.SplitMix64(0x5EED0000 + k).uniform01(24)[13] * 4) % 4 == 2


def sub_voxel_plan(g):
    return g["hs"] < g["sres"] or g["ht"] < g["tres"]


def lattice(k):
    """Draw k puts its points on the half-voxel lattice (mode 3 of draw_case): window edges then fall
    on voxel centres up to the FP32 rounding of the coordinates."""
    return int(synth.SplitMix64(0x5EED0000 + k).uniform01(24)[13] * 4) % 4 == 3


def check_or_report(gpu, ref, what, outside_domain, why, k=None):
    """north_star's bound (1e-5 of the grid's maximum + exact support outside the oracle's 1e-6
    ambiguity band) is REQUIRED inside the engine's stated domain (every bandwidth spans at least one
    voxel; include/stkde.h).  Two KNOWN DEVIATIONS, decided from the inputs alone, are reported as
    xfail with their figures instead of being hidden (DESIGN.md sections 5 and 3.10):
    (1) `outside_domain`: the value bound may be missed; the support must still be exact and the error
        below 1e-3 of the maximum (no gross error);
    (2) lattice draws: the temporal gate is decided in FP32 on the tile-relative position (half an
        ulp = 7.6e-6 voxel on Bt = 128 tiles), wider than the oracle's band, so a pair within ~8e-6
        (relative) of the window edge can be gated the other way; K_t -> 0 there, so the values
        differ by < 1e-6 of the maximum and only the support bit (value > 0) can differ."""
    try:
        assert_parity(gpu, ref.vol, ref.slack, ref.amb, what=what)
    except AssertionError as e:
        lat = k is not None and lattice(k)
        if not (outside_domain or lat):
            raise
        gpu64 = np.asarray(gpu, np.float64)
        vmax = float(ref.vol.max())
        mism = ((gpu64 > 0) != (ref.vol > 0)) & (ref.amb == 0)
        if mism.any():
            assert lat, what + ": support differs"
            edge = float(np.maximum(gpu64[mism], ref.vol[mism]).max())
            assert edge <= 1e-6 * vmax, what + ": support differs at voxels of value %.3e of max" % (edge / vmax)
            why = "FP32 temporal gate at the window edge, %d voxels of value <= %.1e of max" % (int(mism.sum()), edge / vmax)
        rel = float((np.abs(gpu64 - ref.vol) - ref.slack).max() / vmax)
        assert rel <= (1e-3 if outside_domain else 1e-5), what + ": error %.3e of max" % rel
        pytest.xfail("known deviation (%s): max |gpu - oracle| = %.2e of the grid's maximum: %s" % (why, rel, str(e)[:120]))


@pytest.fixture(scope="module")
def S():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1705_09366_b200 as S
    S.load_library()
    return S


@pytest.mark.parametrize("k", range(NCASES))
def test_random_plan_parity(S, oracle_mod, k, monkeypatch):
    g, kernel, pts, cut = draw_case(k)
    monkeypatch.setenv("STKDE_ENGINE", "2")
    if k % 3 == 1:                       # the large grids' tile height on a small grid
        monkeypatch.setenv("STKDE_BT", "128")
    ref = oracle_mod.stkde_pb(pts, kernel=kernel, **g)
    dev = torch.device("cuda", 0)
    with S.Plan(max_n=len(pts), kernel=kernel, device=0, **g) as p:
        info = p.info()
        t = torch.from_numpy(pts).to(dev)
        full = p.compute(t)
        C = int(p.count_contributions(t).item())
        again = p.compute(t)
        torch.cuda.synchronize()
        p.check()
        what = "fuzz %d %s kernel %d n %d engine %s" % (k, g, kernel, len(pts), info.get("engine"))
        assert torch.equal(full, again), what + ": not deterministic"
        gpu = full.cpu().numpy()
        assert C == ref.contributions, what
        # a random time slab and a random x-slab are the full grid's voxels, bitwise
        t0, t1 = sorted((int(cut[0] * (g["Gt"] + 1)), int(cut[1] * (g["Gt"] + 1))))
        if t1 > t0:
            s = p.compute_slab(t, t0, t1, n_norm=len(pts)).cpu().numpy()
            assert np.array_equal(s, gpu[:, :, t0:t1]), what + ": time slab [%d, %d)" % (t0, t1)
        # x cuts are multiples of 16 (the tile width) or G_x (include/stkde.h, stkde_compute_xslab)
        xs = sorted({0, g["Gx"]} | set(range(16, g["Gx"], 16)))
        x0, x1 = sorted((xs[int(cut[2] * len(xs)) % len(xs)], xs[int(cut[3] * len(xs)) % len(xs)]))
        if x1 > x0 and info["engine"] == 2:
            s = p.compute_xslab(t, x0, x1, n_norm=len(pts)).cpu().numpy()
            assert np.array_equal(s, gpu[x0:x1]), what + ": x slab [%d, %d)" % (x0, x1)
        p.check()
    check_or_report(gpu, ref, what, sub_voxel_plan(g), "bandwidth below one voxel", k)


@pytest.mark.parametrize("eng", [1, 0, 3], ids=["mma", "simt", "ws"])
@pytest.mark.parametrize("k", range(0, NCASES, 2))
def test_random_plan_parity_other_engines(S, oracle_mod, k, eng, monkeypatch):
    # the FP32-pipe engines kept beside tcgen05 on the same draws; a plan
    # outside an engine's range falls back (info["engine"] says to which), the result still
    # has to meet the oracle
    g, kernel, pts, _ = draw_case(k)
    monkeypatch.setenv("STKDE_ENGINE", str(eng))
    ref = oracle_mod.stkde_pb(pts, kernel=kernel, **g)
    dev = torch.device("cuda", 0)
    with S.Plan(max_n=len(pts), kernel=kernel, device=0, **g) as p:
        t = torch.from_numpy(pts).to(dev)
        gpu = p.compute(t).cpu().numpy()
        p.check()
        what = "fuzz %d %s kernel %d n %d engine %s (asked %d)" % (k, g, kernel, len(pts), p.info()["engine"], eng)
    # the FP32-accumulating engines add ~N u of rounding on N coincident points (the tcgen05 sums are exact)
    check_or_report(gpu, ref, what, sub_voxel_plan(g) or pile_up(k),
                    "bandwidth below one voxel / FP32 accumulation over a pile-up", k)


def draw_bandwidths(k, g, n):
    """Per-point (hs_i, ht_i) = lambda_i x the plan's, lambda in [0.25, 1] (reading R15), FP32,
    never above the plan's bandwidth; an eighth of the points sit exactly at the cap."""
    from test_gpu_adaptive import f32_le
    v = synth.SplitMix64(0xADA0000 + k).uniform01(2 * n).reshape(-1, 2)
    cap = np.array([f32_le(g["hs"]), f32_le(g["ht"])], np.float32)
    bw = ((0.25 + 0.75 * v) * np.array([g["hs"], g["ht"]])).astype(np.float32)
    bw[: n // 8] = cap
    return np.ascontiguousarray(np.minimum(bw, cap))


def full_scale(oracle_mod, g, kernel, n, bw=None):
    """The largest value one point can add to a voxel: k_s(0, 0) k_t(0) / (n hs_i^2 ht_i) at the
    smallest bandwidths.  The tcgen05 engine's fixed-point factors resolve
    ~8e-7 of THIS per contribution, whatever the grid's maximum turns out to be."""
    if bw is None:
        w = 1.0 / (g["hs"] ** 2 * g["ht"])
    else:
        b = np.asarray(bw, np.float64)
        w = float((1.0 / (b[:, 0] ** 2 * b[:, 1])).max())
    return w * oracle_mod.k_s(0.0, 0.0, kernel) * oracle_mod.k_t(0.0, kernel) / n


def sub_voxel(g, bw):
    """Input-only criterion of the known deviation ('scale of the tolerance'): some
    point's disc or window can miss every voxel centre near its peak, so the grid's maximum may
    lie far below the fixed-point full scale."""
    return float(bw[:, 0].min()) < g["sres"] or float(bw[:, 1].min()) < g["tres"]


@pytest.mark.parametrize("k", range(NCASES))
def test_random_plan_adaptive_parity(S, oracle_mod, k, monkeypatch):
    g, kernel, pts, cut = draw_case(k)
    bw = draw_bandwidths(k, g, len(pts))
    monkeypatch.setenv("STKDE_ENGINE", "2")
    if k % 3 == 2:
        monkeypatch.setenv("STKDE_BT", "128")
    ref = oracle_mod.stkde_pb_adaptive(pts, bw, kernel=kernel, **g)
    dev = torch.device("cuda", 0)
    with S.Plan(max_n=len(pts), kernel=kernel, device=0, **g) as p:
        t = torch.from_numpy(pts).to(dev)
        b = torch.from_numpy(bw).to(dev)
        full = p.compute_adaptive(t, b)
        C = int(p.count_contributions_adaptive(t, b).item())
        gpu = full.cpu().numpy()
        p.check()
        what = "adaptive fuzz %d %s kernel %d n %d" % (k, g, kernel, len(pts))
        assert C == ref.contributions, what
        t0, t1 = sorted((int(cut[0] * (g["Gt"] + 1)), int(cut[1] * (g["Gt"] + 1))))
        if t1 > t0:
            s = p.compute_adaptive_slab(t, b, t0, t1, n_norm=len(pts)).cpu().numpy()
            assert np.array_equal(s, gpu[:, :, t0:t1]), what + ": time slab [%d, %d)" % (t0, t1)
        p.check()
    # sub-voxel per-point bandwidths: the heaviest points may cover no voxel centre, and the grid's
    # maximum is then a pile of contributions far below the fixed-point full scale
    check_or_report(gpu, ref, what, sub_voxel(g, bw), "sub-voxel per-point bandwidth", k)


def contributions_per_voxel(pts, bw, g):
    """Number of (point, voxel) pairs per voxel by the plain definition (strict disc, closed
    window, voxel centres) -- numpy over each point's box, small cases only."""
    nv = np.zeros((g["Gx"], g["Gy"], g["Gt"]), np.int64)
    xc = g["x0"] + (np.arange(g["Gx"]) + 0.5) * g["sres"]
    yc = g["y0"] + (np.arange(g["Gy"]) + 0.5) * g["sres"]
    tc = g["t0"] + (np.arange(g["Gt"]) + 0.5) * g["tres"]
    for (x, y, t), (hs, ht) in zip(np.asarray(pts, np.float64), np.asarray(bw, np.float64)):
        mx = np.flatnonzero(np.abs(xc - x) < hs)
        my = np.flatnonzero(np.abs(yc - y) < hs)
        mt = np.flatnonzero(np.abs(tc - t) <= ht)
        if len(mx) and len(my) and len(mt):
            disc = ((xc[mx] - x)[:, None] ** 2 + (yc[my] - y)[None, :] ** 2) < hs * hs
            nv[np.ix_(mx, my, mt)] += disc[:, :, None].astype(np.int64)
    return nv


def test_single_point_far_below_full_scale(S, oracle_mod):
    # the same regime with a fixed bandwidth, at its smallest: one point on the corner between four
    # voxel centres with h_s = 0.75 voxel; every value on the grid is <= (1 - 2/3)^4 = 1.2 % of
    # the point's peak.  The engine's bound (1e-5 of full scale) holds; the error relative to the
    # grid's own maximum is printed (DESIGN.md §5 quotes it).
    g = dict(x0=0.0, y0=0.0, t0=0.0, sres=1.0, tres=1.0, Gx=20, Gy=20, Gt=20, hs=0.75, ht=3.0)
    pts = np.array([[10.0, 10.0, 10.25]], np.float32)
    ref = oracle_mod.stkde_pb(pts, **g)
    assert ref.contributions == 4 * 6 and ref.amb.sum() == 0
    dev = torch.device("cuda", 0)
    with S.Plan(max_n=1, device=0, **g) as p:
        gpu = p.compute(torch.from_numpy(pts).to(dev)).cpu().numpy()
        p.check()
    fs = full_scale(oracle_mod, g, 0, 1)
    assert float(ref.vol.max()) < 0.013 * fs
    assert_parity(gpu, ref.vol, ref.slack, ref.amb, vmax=fs, what="corner point (engine bound)")
    print("corner point: max |gpu - oracle| = %.3e of full scale, %.3e of the grid's maximum"
          % (np.abs(gpu - ref.vol).max() / fs, np.abs(gpu - ref.vol).max() / ref.vol.max()))


@pytest.mark.parametrize("k", range(0, NCASES, 2))
def test_random_plan_f64_parity(S, oracle_mod, k):
    # the FP64-output option: exact support mask, rtol 2 (n + 2) u
    from test_gpu_f64 import assert_f64_parity, run_f64
    g, kernel, pts, _ = draw_case(k)
    ref = oracle_mod.stkde_pb(pts, kernel=kernel, **g)
    gpu = run_f64(S, pts, kernel=kernel, **g)
    assert_f64_parity(gpu, ref.vol, len(pts), what="f64 fuzz %d %s kernel %d" % (k, g, kernel))
    if k % 4 == 0:
        bw = draw_bandwidths(k, g, len(pts))
        refa = oracle_mod.stkde_pb_adaptive(pts, bw, kernel=kernel, **g)
        gpua = run_f64(S, pts, kernel=kernel, bw=bw, **g)
        assert_f64_parity(gpua, refa.vol, len(pts), what="f64 adaptive fuzz %d %s kernel %d" % (k, g, kernel))


@pytest.mark.parametrize("kernel", [0, 1], ids=["printed", "classical"])
def test_adaptive_scale_never_overflows(S, oracle_mod, kernel):
    # The adaptive full scale is max_i W_i s_i with s_i the point's spatial factor at its nearest
    # voxel column (k_prep): a point whose nearest centre sits just inside its disc edge makes s_i
    # tiny, and W_i / scale * a_x * a_y must still not exceed 1 in the generators' FP32 arithmetic
    # (a fixed-point code above 2^23 - 1 would wrap).  One point per call (it alone sets the
    # scale), u = d / hs_i from 0.5 to 0.99999 at its nearest centre, at tile-relative positions
    # up to 16 + H_s with the plan's H_s = 100; a wrapped code would miss the oracle grossly.
    g = dict(x0=0.0, y0=0.0, t0=0.0, sres=1.0, tres=1.0, Gx=260, Gy=40, Gt=12, hs=100.0, ht=2.0)
    r = synth.SplitMix64(777 + kernel)
    dev = torch.device("cuda", 0)
    worst = 0.0
    with S.Plan(max_n=1, kernel=kernel, device=0, **g) as p:
        for j, u in enumerate([0.5, 0.9, 0.99, 0.999, 0.9999, 0.99999] * 4):
            v = r.uniform01(6)
            X = [0, 15, 16, 127, 143, 259][int(v[0] * 6) % 6]
            Y = int(v[1] * g["Gy"])
            fx, fy = 0.02 + 0.96 * v[2], 0.02 + 0.96 * v[3]
            # distance to the nearest centre in the axis the kernel's factor is evaluated on
            d = max(abs(fx - 0.5), abs(fy - 0.5)) if kernel == 0 else float(np.hypot(fx - 0.5, fy - 0.5))
            hs_i = np.float32(min(max(d / u, 1e-3), 100.0))
            pts = np.array([[X + fx, Y + fy, 5.0 + v[4]]], np.float32)
            bw = np.array([[hs_i, np.float32(0.8 + v[5])]], np.float32)
            ref = oracle_mod.stkde_pb_adaptive(pts, bw, kernel=kernel, **g)
            gpu = p.compute_adaptive(torch.from_numpy(pts).to(dev), torch.from_numpy(bw).to(dev)).cpu().numpy()
            p.check()
            clear = ref.amb == 0
            assert np.array_equal((gpu > 0) & clear, (ref.vol > 0) & clear), (j, u, pts, bw)
            if ref.vol.max() > 0:
                # gross-error check: a wrapped code is off by the full scale, i.e. O(1) of this grid's
                # maximum.  Not the 1e-5 parity bound: at u -> 1 the grid's maximum is (1 - u)^2 or
                # 1 - u^2 ~ 1e-5 of the point's peak, where the FP32 in-voxel fraction alone (2^-24 of
                # a voxel) moves the value by ~1e-3 of itself (measured: 1.8e-3 at
                # u = 0.99999, classical kernel).  The achieved figure is printed.
                e = float((np.abs(gpu - ref.vol) - ref.slack).max() / ref.vol.max())
                worst = max(worst, e)
                assert e <= (1e-5 if u <= 0.99 else 2e-2), (j, u, pts.tolist(), bw.tolist(), e)
    print("adaptive single points near the disc edge: worst |gpu - oracle| / max = %.2e" % worst)
