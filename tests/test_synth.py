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
