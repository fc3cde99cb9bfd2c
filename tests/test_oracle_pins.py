"""Pins for the FP64 oracle against what the paper and mathematics fix.

Each test names the passage it follows and the plausible oracle mistake it
would catch.  None of these retype the oracle's own formula and compare it with
itself: they use printed values (tests/golden/kernel_values.json), closed forms,
invariants, and an independent brute force (Alg. 1 VB vs the point-major PB
loop, plus numpy lattice counting).
"""
import json
import math
import os

import numpy as np
import pytest

import stkde_synth as synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "kernel_values.json")))


def grid(G=(16, 16, 16), res=1.0, hs=3.0, ht=2.0, origin=(0.0, 0.0, 0.0), tres=None):
    return dict(x0=origin[0], y0=origin[1], t0=origin[2], sres=res,
                tres=res if tres is None else tres, Gx=G[0], Gy=G[1], Gt=G[2], hs=hs, ht=ht)


# --------------------------------------------------------------- kernels ---
@pytest.mark.parametrize("kind,kid", [("printed", 0), ("classical", 1)])
def test_kernel_values_match_printed_examples(oracle_mod, kind, kid):
    # PAPER.md:132-133.  Catches a (1-u^2) vs (1-u)^2 swap, a
    # missing pi/2 or 3/4 factor.
    for u, v, want in GOLD[kind]["k_s"]:
        assert oracle_mod.k_s(u, v, kid) == pytest.approx(want, rel=1e-15, abs=1e-15)
    for w, want in GOLD[kind]["k_t"]:
        assert oracle_mod.k_t(w, kid) == pytest.approx(want, rel=1e-15, abs=1e-15)


def test_H_ceil(oracle_mod):
    # PAPER.md:164-166.
    for h, res, want in GOLD["H"]["cases"]:
        assert oracle_mod.H(h, res) == want


def test_mass_constant_by_quadrature():
    # Independent check of the fixture's closed form by numerical
    # quadrature of the printed kernels.
    from scipy import integrate
    kt = integrate.quad(lambda w: 0.75 * (1 - abs(w)) ** 2, -1, 1)[0]
    ks = integrate.dblquad(lambda v, u: math.pi / 2 * (1 - abs(u)) ** 2 * (1 - abs(v)) ** 2,
                           -1, 1, lambda u: -math.sqrt(1 - u * u), lambda u: math.sqrt(1 - u * u))[0]
    assert kt == pytest.approx(0.5, rel=1e-12)
    assert kt * ks == pytest.approx(GOLD["mass"]["printed"], rel=1e-10)


# ------------------------------------------------------- closed forms -----
@pytest.mark.parametrize("kid,expect", [(0, 3 * math.pi / 8), (1, 3 / (2 * math.pi))])
def test_single_point_at_voxel_centre(oracle_mod, kid, expect):
    # n=1, point at a voxel centre -> f = k_s(0,0) k_t(0)/(hs^2 ht).
    # Catches a wrong normalisation (n hs^2 ht) or an off-by-half voxel centre.
    g = grid(G=(17, 15, 13), res=0.5, hs=1.3, ht=0.9)
    p = np.array([[0.5 * 8 + 0.25, 0.5 * 7 + 0.25, 0.5 * 6 + 0.25]], np.float32)
    r = oracle_mod.stkde_pb(p, kernel=kid, **g)
    assert r.vol[8, 7, 6] == pytest.approx(expect / (1.3 ** 2 * 0.9), rel=1e-14)
    assert r.vol.max() == r.vol[8, 7, 6]


@pytest.mark.parametrize("H", [1, 3, 5, 32])
def test_temporal_line_sum_closed_form(oracle_mod, H):
    # Point on a voxel centre with ht = H*tres: sum_T k_t = 0.75 (1 + (H-1)(2H-1)/(3H))
    # (SURVEY §8(c) pin).  Catches a strict-vs-inclusive temporal gate error only
    # via values (edge value is 0), and an abs()/sign error or a window typo
    # (T_i +- H_s instead of +- H_t) via the sum.
    Gt = 2 * H + 5
    g = grid(G=(5, 5, Gt), res=1.0, hs=1.0, ht=float(H))
    c = Gt // 2
    p = np.array([[2.5, 2.5, c + 0.5]], np.float32)
    r = oracle_mod.stkde_pb(p, **g)
    line = r.vol[2, 2, :] * (1.0 * 1.0 * H) / (math.pi / 2)
    want = 0.75 * (1 + (H - 1) * (2 * H - 1) / (3 * H))
    assert line.sum() == pytest.approx(want, rel=1e-13)
    assert np.count_nonzero(line) == 2 * H - 1          # |dt| = ht layers carry value 0


def test_separability_rank_one(oracle_mod):
    # Fig. 3 / PAPER.md:274-289: one point's volume is K_s(X,Y) x K_t(T).
    g = grid(G=(20, 20, 20), res=1.0, hs=6.3, ht=4.7)
    p = np.array([[10.37, 9.81, 10.13]], np.float32)
    v = oracle_mod.stkde_pb(p, **g).vol.reshape(400, 20)
    u, s, _ = np.linalg.svd(v)
    assert s[1] <= 1e-13 * s[0]
    # total = (sum_XY Ks)(sum_T Kt) / (n hs^2 ht), with each factor brute-summed in numpy
    X = np.arange(20) + 0.5
    dx = X[:, None] - np.float64(np.float32(10.37))
    dy = X[None, :] - np.float64(np.float32(9.81))
    d = np.sqrt(dx * dx + dy * dy)
    ks = np.where(d < 6.3, math.pi / 2 * (1 - abs(dx) / 6.3) ** 2 * (1 - abs(dy) / 6.3) ** 2, 0)
    dt = np.abs(X - np.float64(np.float32(10.13)))
    kt = np.where(dt <= 4.7, 0.75 * (1 - dt / 4.7) ** 2, 0)
    assert v.sum() == pytest.approx(ks.sum() * kt.sum() / (6.3 ** 2 * 4.7), rel=1e-12)


@pytest.mark.parametrize("kid,tol", [(0, 2e-3), (1, 5e-4)])
def test_mass_riemann_sum(oracle_mod, kid, tol):
    # Sum f * sres^2 * tres -> integral of the kernels (GOLD mass) for a point
    # whose cylinder spans 32 voxels (SURVEY §8(c) mass pin, D3 bound).
    # Catches a missing 1/n, 1/hs^2 or 1/ht, and a radius-vs-diameter mistake.
    want = GOLD["mass"]["printed" if kid == 0 else "classical"]
    r = synth.SplitMix64(77)
    offs = r.uniform01(6)
    for k in range(3):
        g = grid(G=(70, 70, 70), res=0.25, hs=8.0, ht=8.0)
        p = np.array([[8.5 + 0.25 * offs[2 * k], 8.75 + 0.25 * offs[2 * k + 1], 8.6 + 0.1 * k]],
                     np.float32)
        m = oracle_mod.stkde_pb(p, kernel=kid, with_ambiguity=False, **g).vol.sum() * 0.25 ** 3
        assert abs(m / want - 1) < tol


# ------------------------------------------------------------ invariants ---
def test_mirror_symmetry(oracle_mod):
    # point at the exact grid centre -> volume invariant under
    # X -> Gx-1-X etc.  Catches a signed (u instead of |u|) kernel argument
    # (PAPER.md:132 prints it unsigned) and a corner-sampled voxel.
    for kid in (0, 1):
        g = grid(G=(21, 17, 15), res=1.0, hs=5.5, ht=4.0)
        p = np.array([[10.5, 8.5, 7.5]], np.float32)
        v = oracle_mod.stkde_pb(p, kernel=kid, **g).vol
        assert np.array_equal(v, v[::-1, :, :])
        assert np.array_equal(v, v[:, ::-1, :])
        assert np.array_equal(v, v[:, :, ::-1])


def test_transpose_symmetry(oracle_mod):
    # x <-> y swap on a square grid maps the volume to its XY transpose (up to
    # the rounding order of the k_s product; the gates are symmetric exactly).
    pts = synth.clustered_points(60, 3, 2.0, 2.0, (24, 24, 16), seed=11)
    g = grid(G=(24, 24, 16), res=1.0, hs=4.0, ht=3.0)
    a = oracle_mod.stkde_pb(pts, **g)
    b = oracle_mod.stkde_pb(pts[:, [1, 0, 2]], **g)
    assert np.allclose(a.vol, b.vol.transpose(1, 0, 2), rtol=1e-14, atol=0)
    assert np.array_equal(a.vol > 0, b.vol.transpose(1, 0, 2) > 0)
    assert a.contributions == b.contributions


def test_translation_invariance(oracle_mod):
    # Shifting points and origin by an exact multiple of sres leaves the result
    # bitwise identical (points on a 1/1024 lattice so the shift is exact).
    pts = synth.uniform_points(80, (20, 20, 20), seed=5)
    pts = (np.round(pts * 1024) / 1024).astype(np.float32)
    g = grid(G=(20, 20, 20), res=1.0, hs=3.5, ht=2.5)
    a = oracle_mod.stkde_pb(pts, **g).vol
    sh = pts + np.float32([64, 128, 32])
    g2 = grid(G=(20, 20, 20), res=1.0, hs=3.5, ht=2.5, origin=(64.0, 128.0, 32.0))
    b = oracle_mod.stkde_pb(sh, **g2).vol
    assert np.array_equal(a, b)


def test_linearity(oracle_mod):
    # n f is additive over disjoint point sets (the 1/n of PAPER.md:120 accounted for).
    pts = synth.clustered_points(300, 4, 2.5, 2.0, (24, 20, 18), seed=9)
    g = grid(G=(24, 20, 18), res=1.0, hs=3.2, ht=2.6)
    A, B = pts[:110], pts[110:]
    fa = oracle_mod.stkde_pb(A, **g).vol * len(A)
    fb = oracle_mod.stkde_pb(B, **g).vol * len(B)
    f = oracle_mod.stkde_pb(pts, **g).vol * len(pts)
    assert np.max(np.abs(fa + fb - f)) <= 1e-12 * f.max()


def test_empty_point_set(oracle_mod):
    # n = 0 -> all zeros, no division.
    g = grid(G=(8, 9, 10))
    r = oracle_mod.stkde_pb(np.zeros((0, 3), np.float32), **g)
    assert not r.vol.any() and r.contributions == 0
    v = oracle_mod.stkde_vb(np.zeros((0, 3), np.float32), **g)
    assert not v.vol.any()


# ------------------------------------------------ brute force: VB == PB ----
CASES = [
    # (n, G, res, hs, ht, kernel, clustered)
    (0, (16, 16, 16), 1.0, 3.0, 2.0, 0, False),
    (1, (16, 16, 16), 1.0, 3.0, 2.0, 0, False),
    (100, (16, 16, 16), 1.0, 4.0, 3.0, 0, True),
    (200, (20, 18, 22), 0.5, 1.7, 1.1, 0, True),
    (150, (24, 16, 12), 1.0, 2.5, 4.0, 1, False),
    (120, (32, 32, 20), 1.0 / 64, 3.0 / 64, 2.0 / 64, 0, True),
]


@pytest.mark.parametrize("case", CASES)
def test_pb_equals_vb_bitwise(oracle_mod, case):
    # Alg. 1 (VB) written out brute force vs the point-major
    # loop of Alg. 2/3: same per-voxel sum order, so bitwise equal.  Catches
    # loop-bound mistakes in the box (T_i +- H_s typo), clipping
    # errors at the grid faces, and missed points whose box overlaps the grid
    # from outside.  Also checks the contribution counter and ambiguity output.
    n, G, res, hs, ht, kid, clustered = case
    ext = (G[0] * res, G[1] * res, G[2] * res)
    if clustered:
        pts = synth.clustered_points(n, 3, 3 * res, 3 * res, ext, seed=n + 3)
    else:
        pts = synth.uniform_points(n, ext, seed=n + 4)
    # a few points just outside the box (cylinder reaches inside; reading R6)
    if n >= 100:
        pts = np.concatenate([pts, np.array([[-1.5 * res, ext[1] / 2, ext[2] / 2],
                                             [ext[0] + 0.7 * res, 0.3 * res, ext[2] + 0.5 * res]],
                                            np.float32)])
    g = grid(G=G, res=res, hs=hs, ht=ht)
    vb = oracle_mod.stkde_vb(pts, kernel=kid, **g)
    pb1 = oracle_mod.stkde_pb(pts, kernel=kid, nthreads=1, **g)
    pb4 = oracle_mod.stkde_pb(pts, kernel=kid, nthreads=4, **g)
    assert np.array_equal(vb.vol, pb1.vol)
    assert np.array_equal(pb1.vol, pb4.vol)
    assert np.array_equal(vb.amb, pb1.amb)
    assert np.allclose(vb.slack, pb1.slack, rtol=1e-12, atol=0)
    assert vb.contributions == pb1.contributions == pb4.contributions
    assert vb.contributions == oracle_mod.contributions(pts, kernel=kid, **g)
    if kid == 0:
        assert (pb1.vol >= 0).all()


def test_contributions_lattice_count(oracle_mod):
    # C for one interior point on a voxel centre = (#lattice points strictly
    # inside radius r) x (2H_t+1), counted here by numpy enumeration.
    for r_, Ht in [(3, 1), (5, 4), (8, 2)]:
        G = 2 * r_ + 5
        g = grid(G=(G, G, 2 * Ht + 5), res=1.0, hs=float(r_), ht=float(Ht))
        p = np.array([[G // 2 + 0.5, G // 2 + 0.5, Ht + 2.5]], np.float32)
        k = np.arange(-r_ - 1, r_ + 2)
        disc = int(((k[:, None] ** 2 + k[None, :] ** 2) < r_ * r_).sum())
        assert oracle_mod.contributions(p, **g) == disc * (2 * Ht + 1)
        assert oracle_mod.stkde_pb(p, **g).contributions == disc * (2 * Ht + 1)
    assert disc == 197 - 4  # Gauss circle N(8) = 197 (<=), minus the 4 points on x^2+y^2 = 64


def test_gate_edges_and_ambiguity(oracle_mod):
    # Alg. 1 gates: strict spatial, inclusive temporal.
    # Point at voxel centre (5.5, 5.5, 5.5), hs = 3 exactly: voxel X=8 (dx = 3)
    # is outside (strict) but flagged ambiguous; ht = 2: layer T=7/3 (|dt| = 2)
    # is inside with value 0 and ambiguous.
    g = grid(G=(12, 12, 12), res=1.0, hs=3.0, ht=2.0)
    p = np.array([[5.5, 5.5, 5.5]], np.float32)
    r = oracle_mod.stkde_pb(p, **g)
    assert r.vol[8, 5, 5] == 0 and r.amb[8, 5, 5] == 1
    assert r.vol[7, 5, 5] > 0 and r.amb[7, 5, 5] == 0
    assert r.vol[5, 5, 7] == 0 and r.amb[5, 5, 7] == 1 and r.amb[5, 5, 6] == 0
    assert r.contributions == 25 * 5   # 25 disc columns (r = 3, strict) x 5 layers


def test_sampled_voxels_match_full_grid(oracle_mod):
    # Alg. 1 at sampled voxels == the full-grid point-major oracle (bitwise).
    w = synth.make_config("dengue")
    g = w.grid_kwargs()
    full = oracle_mod.stkde_pb(w.points, with_ambiguity=True, **g)
    rng = synth.SplitMix64(3)
    nz = np.flatnonzero(full.vol)
    vox = np.concatenate([nz[(rng.uniform01(200) * len(nz)).astype(np.int64) % len(nz)],
                          (rng.uniform01(50) * full.vol.size).astype(np.int64)])
    val, slack, amb = oracle_mod.stkde_vb_voxels(w.points, vox, **g)
    assert np.array_equal(val, full.vol.reshape(-1)[vox])
    assert np.array_equal(amb, full.amb.reshape(-1)[vox])


def test_tiny_config_full(oracle_mod):
    # The tiny config (BASELINE.json configs[0]) against VB brute force on a
    # 32^3 crop of its grid (the same points, hs = ht = 3/64).
    w = synth.make_config("tiny")
    g = w.grid_kwargs()
    g.update(Gx=32, Gy=32, Gt=32)
    vb = oracle_mod.stkde_vb(w.points[:400], **g)
    pb = oracle_mod.stkde_pb(w.points[:400], **g)
    assert np.array_equal(vb.vol, pb.vol)


# ----------------------------------------------------------------- slack ---
@pytest.mark.parametrize("kid", [0, 1])
def test_slack_closed_form(oracle_mod, kid):
    # Reading R10/R11: slack(voxel) = sum over the voxel's ambiguous pairs
    # of |k_s k_t| / (n hs^2 ht); 0 on unambiguous voxels.  One point at the voxel centre
    # (10.5, 10.5, 10.5), hs = 5, ht = 2 (n = 1):
    #  * columns at integer offsets (3, 4) / (4, 3) lie exactly on the circle d = hs
    #    (Pythagorean): ambiguous, outside the strict gate, k_s(0.6, 0.8) =
    #    pi/2 (0.4)^2 (0.2)^2 = 0.0064 pi/2 printed, 2/pi (1 - 0.36 - 0.64) = 0 classical
    #    (up to the FP64 rounding of 0.6 and 0.8);
    #  * columns (5, 0) / (0, 5): ambiguous, k_s(1, 0) = 0;
    #  * layers dt = +-2 = ht: inside the inclusive temporal gate, ambiguous, k_t(1) = 0.
    # So the slack of a (3,4)-type voxel at layer offset dt is k_s(0.6,0.8) k_t(|dt|/2) / 50,
    # the sum over the grid is 8 k_s(0.6,0.8) (k_t(0) + 2 k_t(0.5)) / 50 = 8 k_s 1.125 / 50,
    # and the ambiguous voxels are the 12 circle columns x 5 layers plus the strict disc
    # interior (Gauss count) x 2 edge layers.  Catches slack = 0 everywhere (a dropped
    # slack), slack added to unambiguous voxels, a missing 1/(n hs^2 ht), or an ambiguity
    # test on the wrong side of the gate.
    g = grid(G=(21, 21, 21), res=1.0, hs=5.0, ht=2.0)
    r = oracle_mod.stkde_pb(np.array([[10.5, 10.5, 10.5]], np.float32), kernel=kid, **g)
    ks34 = (math.pi / 2) * 0.4 ** 2 * 0.2 ** 2 if kid == 0 else 0.0
    kt = {0: 0.75, 1: 0.75 * 0.25 if kid == 0 else 0.75 * 0.75, 2: 0.0}
    for dx, dy in ((3, 4), (-4, 3), (4, -3), (-3, -4)):
        for dt in (-2, -1, 0, 1, 2):
            v = (10 + dx, 10 + dy, 10 + dt)
            assert r.amb[v] == 1 and r.vol[v] == 0
            assert r.slack[v] == pytest.approx(ks34 * kt[abs(dt)] / 50.0, rel=1e-12, abs=1e-16)
    assert r.slack[15, 10, 10] == 0 and r.amb[15, 10, 10] == 1          # k_s(1, 0) = 0
    assert r.slack[10, 10, 12] == 0 and r.amb[10, 10, 12] == 1          # k_t(1) = 0
    assert (r.slack[r.amb == 0] == 0).all() and (r.slack >= 0).all()
    assert r.slack.sum() == pytest.approx(8 * ks34 * (kt[0] + 2 * kt[1]) / 50.0, rel=1e-12, abs=1e-15)
    i, j = np.meshgrid(np.arange(-6, 7), np.arange(-6, 7))
    interior = int((i * i + j * j < 25).sum())
    assert int(r.amb.sum()) == 12 * 5 + interior * 2


def test_slack_edge_jump_bound(oracle_mod):
    # On random inputs every ambiguous pair is within 1e-6 (relative) of an edge, so its
    # |k_s k_t| is at most the printed kernel's edge value: spatial edge (pi/2)(1 - 1/sqrt2)^4
    # = 0.011560 (the maximum of k_s on the unit circle, up to 1e-5 for the 1e-6
    # band) times k_t <= 3/4; temporal edge k_t <= 3/4 (1e-6)^2.  A voxel's slack is bounded
    # by (its ambiguous pair count) x that / (n hs^2 ht); with points on a lattice of voxel
    # centres and integer hs, ht the ambiguous pairs of a voxel are the lattice points at
    # exact distance hs (or exact |dt| = ht), counted here by integer geometry.
    g = grid(G=(24, 24, 16), res=1.0, hs=5.0, ht=2.0)
    rng = synth.SplitMix64(7)
    n = 60
    P = np.stack([np.floor(rng.uniform(0, 24, n)), np.floor(rng.uniform(0, 24, n)),
                  np.floor(rng.uniform(0, 16, n))], axis=1)
    pts = (P + 0.5).astype(np.float32)
    r = oracle_mod.stkde_pb(pts, **g)
    X, Y, T = np.meshgrid(np.arange(24), np.arange(24), np.arange(16), indexing="ij")
    m = np.zeros(X.shape, np.int64)
    for px, py, pt in P.astype(np.int64):
        d2 = (X - px) ** 2 + (Y - py) ** 2
        dt = np.abs(T - pt)
        m += ((d2 == 25) & (dt <= 2)) | ((d2 <= 25) & (dt == 2))
    edge = (math.pi / 2) * (1 - 1 / math.sqrt(2)) ** 4
    bound = m * (edge * (1 + 1e-5) * 0.75) / (n * 25 * 2)
    assert (r.slack <= bound + 1e-300).all()
    assert ((m > 0) == (r.amb == 1)).all()
    assert r.slack.max() > 0
