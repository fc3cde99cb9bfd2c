"""Input generator checks (stkde_synth): SplitMix64 test vectors, determinism, frozen hashes."""
import json
import os

import numpy as np
import pytest

import stkde_synth as synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "synth_sha256.json")))


def test_splitmix64_reference_vectors():
    # Published SplitMix64 outputs (Steele, Lea, Flood 2014 reference stream).
    assert [int(x) for x in synth.SplitMix64(0).next_u64(3)] == [
        0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    assert int(synth.SplitMix64(1234567).next_u64(1)[0]) == 6457827717110365317


def test_counter_form_matches_sequential():
    r = synth.SplitMix64(42)
    a = np.concatenate([r.next_u64(5), r.next_u64(7)])
    assert np.array_equal(a, synth.SplitMix64(42).next_u64(12))


def test_uniform01_range():
    u = synth.SplitMix64(3).uniform01(100000)
    assert u.min() > 0 and u.max() <= 1.0


@pytest.mark.parametrize("name", ["tiny", "dengue", "social", "stress"])
def test_config_frozen_and_in_box(name):
    w = synth.make_config(name)
    g = GOLD[name]
    assert w.n == g["n"] and list(w.G) == g["G"]
    assert synth.points_sha256(w.points) == g["sha256"]
    ext = np.array([w.G[0] * w.sres, w.G[1] * w.sres, w.G[2] * w.tres], np.float32)
    assert (w.points >= 0).all() and (w.points < ext).all()
    assert w.points.dtype == np.float32 and w.points.flags.c_contiguous


@pytest.mark.slow
def test_ornith_frozen():
    w = synth.make_config("ornith")
    assert synth.points_sha256(w.points) == GOLD["ornith"]["sha256"]


@pytest.mark.parametrize("name", ["dengue", "social", "stress"])
def test_adaptive_bandwidths_recipe(name):
    # the bench's adaptive-variant inputs: float32 [n, 2], inside the
    # plan's range (0.25 h .. h, never above the plan's FP64 h), one factor for both
    # axes, deterministic, and narrower where points are dense
    w = synth.make_config(name)
    bw = synth.adaptive_bandwidths(w)
    assert bw.dtype == np.float32 and bw.shape == (w.n, 2) and bw.flags.c_contiguous
    hs, ht = bw[:, 0].astype(np.float64), bw[:, 1].astype(np.float64)
    assert (hs <= w.hs).all() and (ht <= w.ht).all()
    assert (hs >= 0.25 * w.hs * (1 - 1e-6)).all() and (ht >= 0.25 * w.ht * (1 - 1e-6)).all()
    np.testing.assert_allclose(hs / w.hs, ht / w.ht, rtol=1e-6)
    assert np.array_equal(bw, synth.adaptive_bandwidths(w))
    assert hs.min() < hs.max()                      # the recipe actually adapts
    # dense cells get the narrow kernels: mean lambda of the densest decile < sparsest decile
    p = w.points.astype(np.float64)
    cell = np.floor(p / np.array([w.hs, w.hs, w.ht])).astype(np.int64)
    _, inv, cnt = np.unique(cell, axis=0, return_inverse=True, return_counts=True)
    c = cnt[inv.reshape(-1)]
    lo, hi = np.quantile(c, [0.1, 0.9])
    assert hs[c >= hi].mean() < hs[c <= lo].mean()


def test_sweep_fractions():
    f = synth.SWEEP_FRACTIONS
    assert f[0] == 1.0 and all(0 < a <= 1 for a in f) and list(f) == sorted(f, reverse=True)
