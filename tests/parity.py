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


def oracle_xchunks(oracle_mod, points, g, rows, kernel=0):
    """The FP64 oracle (oracle.stkde_pb) over the full grid in X-row chunks [a, b).

    A chunk is the same grid with origin x0 + a*sres and Gx = b - a (host memory: the
    oracle's vol + slack + amb take 17 B per voxel).  Exactness: every voxel centre of the
    chunk, x0' + (X' + 0.5) sres, is checked to be the same FP64 number as the full grid's
    x0 + (a + X' + 0.5) sres (the oracle's centre expression, reading R5), so the chunk's
    gates and kernel values -- hence its sums -- are bitwise the full grid's (the translation
    invariance pin of tests/test_oracle_pins.py in its exact-arithmetic form).
    Yields (a, b, OracleResult)."""
    Gx = int(g["Gx"])
    for a in range(0, Gx, rows):
        b = min(Gx, a + rows)
        x0c = g["x0"] + a * g["sres"]
        X = np.arange(b - a, dtype=np.float64)
        full = g["x0"] + (X + a + 0.5) * g["sres"]
        part = x0c + (X + 0.5) * g["sres"]
        assert np.array_equal(full, part), "X-chunk origin shift is not exact for this grid"
        gc = dict(g, x0=x0c, Gx=b - a)
        yield a, b, oracle_mod.stkde_pb(points, kernel=kernel, **gc)


class DecileReport:
    """Relative error |gpu - oracle| / oracle by oracle-value decile over the support
    (unambiguous voxels with oracle > 0), from every `stride`-th support voxel of each
    chunk (a deterministic sample); reported, not asserted (the acceptance bound is the
    absolute 1e-5 * max of assert_parity)."""

    def __init__(self, stride=97):
        self.stride = stride
        self.vals, self.rels = [], []

    def add(self, gpu, vol, amb):
        m = (vol > 0) & (amb == 0)
        v = vol[m][:: self.stride]
        r = np.abs(np.asarray(gpu, np.float64)[m][:: self.stride] - v) / v
        self.vals.append(v)
        self.rels.append(r)

    def table(self):
        if not self.vals:
            return []
        v = np.concatenate(self.vals)
        r = np.concatenate(self.rels)
        if len(v) == 0:
            return []
        edges = np.quantile(v, np.linspace(0, 1, 11))
        out = []
        for i in range(10):
            sel = (v >= edges[i]) & ((v < edges[i + 1]) if i < 9 else (v <= edges[i + 1]))
            if sel.any():
                out.append((i + 1, float(edges[i]), float(edges[i + 1]), int(sel.sum()),
                            float(np.median(r[sel])), float(r[sel].max())))
        return out

    def format(self, vmax):
        rows = ["decile  value range (/max)          samples   median rel   max rel"]
        for d, lo, hi, k, med, mx in self.table():
            rows.append("%6d  [%.2e, %.2e]   %8d   %.2e     %.2e" % (d, lo / vmax, hi / vmax, k, med, mx))
        return "\n".join(rows)


def cylinder_voxels(points, g, rng, npts=400, per=8, nrand=400):
    """Voxels sampled without looking at the GPU output: `per` random voxels of the box
    X_i +- H_s, Y_i +- H_s, T_i +- H_t (Alg. 2/3 loop bounds) of each of
    `npts` random input points, plus `nrand` uniform voxels.  Linear indices (X*Gy+Y)*Gt+T."""
    n = len(points)
    Hs = int(np.ceil(g["hs"] / g["sres"]))
    Ht = int(np.ceil(g["ht"] / g["tres"]))
    idx = (rng.uniform01(npts) * n).astype(np.int64) % n
    p = np.asarray(points, np.float64)[idx]
    X = np.floor((p[:, 0] - g["x0"]) / g["sres"]).astype(np.int64)
    Y = np.floor((p[:, 1] - g["y0"]) / g["sres"]).astype(np.int64)
    T = np.floor((p[:, 2] - g["t0"]) / g["tres"]).astype(np.int64)
    m = npts * per
    dx = np.rint((rng.uniform01(m) * 2 - 1) * Hs).astype(np.int64)
    dy = np.rint((rng.uniform01(m) * 2 - 1) * Hs).astype(np.int64)
    dt = np.rint((rng.uniform01(m) * 2 - 1) * Ht).astype(np.int64)
    k = np.repeat(np.arange(npts), per)
    Xv = np.clip(X[k] + dx, 0, g["Gx"] - 1)
    Yv = np.clip(Y[k] + dy, 0, g["Gy"] - 1)
    Tv = np.clip(T[k] + dt, 0, g["Gt"] - 1)
    vox = (Xv * g["Gy"] + Yv) * g["Gt"] + Tv
    rnd = (rng.uniform01(nrand) * (g["Gx"] * g["Gy"] * g["Gt"])).astype(np.int64)
    return np.unique(np.concatenate([vox, rnd]))
