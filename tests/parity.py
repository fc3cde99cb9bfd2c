"""Helpers for GPU-vs-oracle parity (tests only).

Acceptance (BASELINE.json north_star, made concrete in DESIGN.md §5):
  * |gpu - oracle| <= 1e-5 * max(oracle) + slack(voxel) everywhere, where
    slack is the oracle's sum of |contribution| over pairs within 1e-6
    (relative) of a bandwidth boundary (0 for unambiguous voxels);
  * the support masks (value > 0) agree exactly outside the ambiguous voxels.
"""
import numpy as np

REL_TOL = 1e-5


def assert_parity(gpu: np.ndarray, vol: np.ndarray, slack: np.ndarray, amb: np.ndarray, vmax=None, what=""):
    gpu = np.asarray(gpu, dtype=np.float64)
    vmax = float(vol.max()) if vmax is None else float(vmax)
    tol = REL_TOL * vmax
    diff = np.abs(gpu - vol)
    bad = diff > tol + slack
    if bad.any():
        idx = np.argwhere(bad)[:5]
        raise AssertionError("%s: %d voxels exceed tol %.3e (max diff %.3e); first %s gpu=%s ref=%s"
                             % (what, int(bad.sum()), tol, float(diff.max()), idx.tolist(),
                                gpu[bad][:5].tolist(), vol[bad][:5].tolist()))
    clear = amb == 0
    sm = (gpu > 0) != (vol > 0)
    sm &= clear
    if sm.any():
        idx = np.argwhere(sm)[:5]
        raise AssertionError("%s: support mask differs at %d unambiguous voxels, first %s gpu=%s ref=%s"
                             % (what, int(sm.sum()), idx.tolist(), gpu[sm][:5].tolist(), vol[sm][:5].tolist()))
    return float(diff.max()) / max(vmax, 1e-300)
