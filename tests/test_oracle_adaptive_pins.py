"""Pins for the adaptive-bandwidth oracle (reading R15).

The adaptive estimator moves h_s, h_t of PAPER.md:120-121 inside the sum, one
pair per point (the "bandwidth that adapts to the density of population" of
PAPER.md:1060-1062).  These tests pin oracle.stkde_*_adaptive against things
other than itself: closed forms, the fixed-bandwidth oracle (pinned in
test_oracle_pins.py) applied point by point, the VB brute force, and the
kernel mass constant.  A mistake such as using the plan's h instead of the
point's, swapping hs_i and ht_i, dropping the per-point 1/(hs_i^2 ht_i), or
clipping the loops at the plan's H instead of the point's, fails one of them.
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


def random_case(seed, n, G, hs, ht, lo=0.3):
    r = synth.SplitMix64(seed)
    u = r.uniform01(3 * n).reshape(n, 3)
    pts = (u * np.array(G, np.float64)).astype(np.float32)
    v = r.uniform01(2 * n).reshape(n, 2)
    bw = np.empty((n, 2), np.float32)
    bw[:, 0] = (lo + (1 - lo) * v[:, 0]) * hs
    bw[:, 1] = (lo + (1 - lo) * v[:, 1]) * ht
    cap = np.array([f32_le(hs), f32_le(ht)], np.float32)   # largest float32 <= the plan's h
    bw[: n // 8] = cap          # some points at the plan maximum
    return pts, np.minimum(bw, cap)


def f32_le(h):
    c = np.float32(h)
    return c if float(c) <= h else np.nextafter(c, np.float32(0))


@pytest.mark.parametrize("kid,k0", [(0, 3 * math.pi / 8), (1, 3 / (2 * math.pi))])
def test_single_point_own_bandwidth_closed_form(oracle_mod, kid, k0):
    # n = 1, point on a voxel centre, its own (hs_i, ht_i) below the plan's:
    # f = k_s(0,0) k_t(0) / (hs_i^2 ht_i) (SPEC.md:155 with h -> h_i).  Catches the
    # plan's h used in the norm or in the gates.
    g = grid(G=(21, 19, 17), res=0.5, hs=3.0, ht=2.5)
    p = np.array([[0.5 * 10 + 0.25, 0.5 * 9 + 0.25, 0.5 * 8 + 0.25]], np.float32)
    bw = np.array([[1.3, 0.9]], np.float32)
    r = oracle_mod.stkde_pb_adaptive(p, bw, kernel=kid, **g)
    hs_i, ht_i = float(np.float32(1.3)), float(np.float32(0.9))
    assert r.vol[10, 9, 8] == pytest.approx(k0 / (hs_i ** 2 * ht_i), rel=1e-14)
    assert r.vol.max() == r.vol[10, 9, 8]
    # support = the point's own cylinder: |dx| < 1.3 -> within 2 voxels (res 0.5), |dt| <= 0.9 -> 1 layer
    nz = np.argwhere(r.vol > 0)
    assert nz[:, 0].min() == 8 and nz[:, 0].max() == 12
    assert nz[:, 2].min() == 7 and nz[:, 2].max() == 9


@pytest.mark.parametrize("kid", [0, 1])
def test_superposition_of_fixed_bandwidth_runs(oracle_mod, kid):
    # n f_adaptive = sum_i f_fixed(point i alone, h = h_i, n = 1): each point's
    # cylinder is the fixed-bandwidth oracle's with its own h.
    G = (18, 14, 12)
    g = grid(G=G, res=1.0, hs=4.0, ht=3.0)
    pts, bw = random_case(5, 24, G, 4.0, 3.0, lo=0.2)
    r = oracle_mod.stkde_pb_adaptive(pts, bw, kernel=kid, with_ambiguity=False, **g)
    acc = np.zeros(G)
    for i in range(len(pts)):
        gi = dict(g, hs=float(bw[i, 0]), ht=float(bw[i, 1]))
        acc += oracle_mod.stkde_pb(pts[i:i + 1], kernel=kid, with_ambiguity=False, **gi).vol
    np.testing.assert_allclose(r.vol * len(pts), acc, rtol=1e-13, atol=1e-16)
    # uniform bandwidths = the plan's: the adaptive estimator is the paper's
    bw_u = np.tile(np.array([[4.0, 3.0]], np.float32), (len(pts), 1))
    ru = oracle_mod.stkde_pb_adaptive(pts, bw_u, kernel=kid, with_ambiguity=False, **g)
    rf = oracle_mod.stkde_pb(pts, kernel=kid, with_ambiguity=False, **g)
    np.testing.assert_allclose(ru.vol, rf.vol, rtol=1e-14, atol=1e-18)


@pytest.mark.parametrize("seed,G,res,hs,ht", [(11, (12, 10, 9), 1.0, 3.0, 2.0),
                                              (12, (9, 11, 13), 0.5, 1.7, 1.1)])
def test_pb_equals_vb_bitwise(oracle_mod, seed, G, res, hs, ht):
    # Alg. 1 (VB) brute force over every voxel and point vs the point-major loop.
    g = grid(G=G, res=res, hs=hs, ht=ht)
    pts, bw = random_case(seed, 60, tuple(x * res for x in G), hs, ht, lo=0.1)
    a = oracle_mod.stkde_pb_adaptive(pts, bw, **g)
    b = oracle_mod.stkde_vb_adaptive(pts, bw, **g)
    assert np.array_equal(a.vol, b.vol)
    assert np.array_equal(a.amb, b.amb)
    np.testing.assert_allclose(a.slack, b.slack, rtol=1e-14, atol=0)
    assert a.contributions == b.contributions
    assert oracle_mod.contributions_adaptive(pts, bw, **g) == a.contributions
    # sampled voxels = the full grid at those voxels (same per-voxel order)
    r = synth.SplitMix64(seed + 100)
    vox = (r.uniform01(40) * (G[0] * G[1] * G[2])).astype(np.int64)
    val, _, amb = oracle_mod.stkde_vb_voxels_adaptive(pts, bw, vox, **g)
    assert np.array_equal(val, a.vol.reshape(-1)[vox])
    assert np.array_equal(amb, a.amb.reshape(-1)[vox])


def test_contributions_equal_sum_of_fixed_counts(oracle_mod):
    G = (20, 20, 16)
    g = grid(G=G, res=1.0, hs=5.0, ht=4.0)
    pts, bw = random_case(21, 30, G, 5.0, 4.0, lo=0.15)
    want = sum(oracle_mod.contributions(pts[i:i + 1], **dict(g, hs=float(bw[i, 0]), ht=float(bw[i, 1])))
               for i in range(len(pts)))
    assert oracle_mod.contributions_adaptive(pts, bw, **g) == want


def test_mass_per_point(oracle_mod):
    # Each point carries the printed kernels' mass whatever its bandwidth
    # (SURVEY D3 constant, Riemann bound at >= 30 voxels of radius).
    want = GOLD["mass"]["printed"]
    g = grid(G=(72, 72, 72), res=0.25, hs=8.0, ht=8.0)
    p = np.array([[9.1, 8.85, 9.0], [9.3, 9.05, 8.7]], np.float32)
    bw = np.array([[8.0, 7.5], [7.5, 8.0]], np.float32)
    m = oracle_mod.stkde_pb_adaptive(p, bw, with_ambiguity=False, **g).vol.sum() * 0.25 ** 3
    assert abs(m / want - 1) < 2e-3


def test_bandwidth_above_plan_rejected(oracle_mod):
    g = grid()
    p = np.array([[5.0, 5.0, 5.0]], np.float32)
    with pytest.raises(ValueError):
        oracle_mod.stkde_pb_adaptive(p, np.array([[3.5, 1.0]], np.float32), **g)
    with pytest.raises(ValueError):
        oracle_mod.stkde_pb_adaptive(p, np.array([[1.0, 0.0]], np.float32), **g)
