"""Seeded synthetic STKDE workloads shared by the oracle tests and the GPU path.

This module is INPUT PLUMBING ONLY: it draws point clouds and names grid
parameters.  It holds none of the method's arithmetic (no kernels, no gates,
no voxel mapping, no normalisation), so that `oracle/` and the CUDA path can
both consume its output while sharing no code with each other.

Generator (SPEC.md:439-447 / 471 "io: generate_synthetic"):
  * PRNG: SplitMix64 in its counter form, state_k = seed + k*GAMMA, out = mix(state_k)
    (identical to the sequential SplitMix64 stream), vectorised in numpy uint64.
  * u64 -> (0,1]: (x >> 11) * 2^-53, with 0 mapped to 2^-53.
  * Normals: Box-Muller on two (0,1] uniforms.
  * Zipf(a) over K categories: weights k^-a, sampled by inverse CDF.
  * Points are generated in FP64, rounded once to FP32 and clamped into the
    half-open box [0, extent) per axis (FP32 nextafter below the upper edge).

The five BASELINE.json configs stand in for the paper's Table 2 datasets
(PAPER.md:606-687), which are not available: tiny, dengue-like (Dengue,
PAPER.md:608-619), social-media-like (PollenUS),
ornithology-like (eBird) and the large-bandwidth stress
instance (PollenUS_Hr-Hb / Dengue_Hr-VHb).
"""
from __future__ import annotations

import dataclasses
import hashlib

import numpy as np

__all__ = ["SplitMix64", "Workload", "CONFIGS", "make_config", "points_sha256",
           "uniform_points", "clustered_points"]

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_TWO_M53 = 2.0 ** -53


def _mix(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


class SplitMix64:
    """Counter-form SplitMix64: draw k of the stream is mix(seed + (k+1)*GAMMA)."""

    def __init__(self, seed: int):
        self._state = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)

    def next_u64(self, m: int) -> np.ndarray:
        ctr = np.arange(1, m + 1, dtype=np.uint64)
        with np.errstate(over="ignore"):
            z = self._state + ctr * _GAMMA
            self._state = np.uint64(self._state + np.uint64(m) * _GAMMA)
        return _mix(z)

    def uniform01(self, m: int) -> np.ndarray:
        """m draws in (0,1] (SPEC.md:471 mapping)."""
        x = self.next_u64(m) >> np.uint64(11)
        u = x.astype(np.float64) * _TWO_M53
        u[x == 0] = _TWO_M53
        return u

    def uniform(self, lo, hi, m: int) -> np.ndarray:
        u = self.uniform01(m)
        return lo + (1.0 - u) * (hi - lo)  # (0,1] -> [lo, hi)

    def normal(self, m: int) -> np.ndarray:
        u1 = self.uniform01(m)
        u2 = self.uniform01(m)
        return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)

    def categorical(self, weights, m: int) -> np.ndarray:
        w = np.asarray(weights, dtype=np.float64)
        cdf = np.cumsum(w) / w.sum()
        idx = np.searchsorted(cdf, self.uniform01(m), side="left")
        return np.minimum(idx, len(w) - 1)

    def zipf_weights(self, a: float, k: int) -> np.ndarray:
        return np.arange(1, k + 1, dtype=np.float64) ** (-a)

    def permutation(self, m: int) -> np.ndarray:
        return np.argsort(self.next_u64(m), kind="stable")


@dataclasses.dataclass(frozen=True)
class Workload:
    """A point set plus the grid it is estimated on (world units)."""

    name: str
    points: np.ndarray          # float32 [n, 3]: x, y, t
    origin: tuple               # (x0, y0, t0)
    sres: float
    tres: float
    G: tuple                    # (Gx, Gy, Gt)
    hs: float
    ht: float

    @property
    def n(self) -> int:
        return int(self.points.shape[0])

    def grid_kwargs(self) -> dict:
        return dict(x0=self.origin[0], y0=self.origin[1], t0=self.origin[2],
                    sres=self.sres, tres=self.tres, Gx=self.G[0], Gy=self.G[1],
                    Gt=self.G[2], hs=self.hs, ht=self.ht)


def _clamp_f32(v: np.ndarray, lo: float, hi: float) -> np.ndarray:
    """Round FP64 -> FP32 once, then clamp into [lo, hi) in FP32."""
    f = v.astype(np.float32)
    f = np.maximum(f, np.float32(lo))
    top = np.nextafter(np.float32(hi), np.float32(-np.inf), dtype=np.float32)
    return np.minimum(f, top)


def _pack(x, y, t, extent) -> np.ndarray:
    pts = np.empty((len(x), 3), dtype=np.float32)
    pts[:, 0] = _clamp_f32(np.asarray(x), 0.0, extent[0])
    pts[:, 1] = _clamp_f32(np.asarray(y), 0.0, extent[1])
    pts[:, 2] = _clamp_f32(np.asarray(t), 0.0, extent[2])
    return pts


def uniform_points(n: int, extent, seed: int) -> np.ndarray:
    """n points uniform in [0,extent) (test helper; no method arithmetic)."""
    r = SplitMix64(seed)
    return _pack(r.uniform(0, extent[0], n), r.uniform(0, extent[1], n),
                 r.uniform(0, extent[2], n), extent)


def clustered_points(n: int, clusters: int, sigma_xy: float, sigma_t: float,
                     extent, seed: int) -> np.ndarray:
    """SPEC.md io.generate_synthetic: uniform centres, uniform cluster choice, Box-Muller offsets."""
    r = SplitMix64(seed)
    cx = r.uniform(0, extent[0], clusters)
    cy = r.uniform(0, extent[1], clusters)
    ct = r.uniform(0, extent[2], clusters)
    k = r.categorical(np.ones(clusters), n)
    return _pack(cx[k] + sigma_xy * r.normal(n), cy[k] + sigma_xy * r.normal(n),
                 ct[k] + sigma_t * r.normal(n), extent)


# ---------------------------------------------------------------- configs ---

def _tiny(seed=1):
    # BASELINE.json configs[0]: n=2000 in [0,1]^3; 70% from 5 isotropic Gaussians
    # (sigma 0.05 space, 0.08 time), 30% uniform; 64^3 grid; hs = ht = 3 voxels.
    r = SplitMix64(seed)
    n, nc = 2000, 1400
    cx, cy, ct = r.uniform(0, 1, 5), r.uniform(0, 1, 5), r.uniform(0, 1, 5)
    k = r.categorical(np.ones(5), nc)
    x = np.concatenate([cx[k] + 0.05 * r.normal(nc), r.uniform(0, 1, n - nc)])
    y = np.concatenate([cy[k] + 0.05 * r.normal(nc), r.uniform(0, 1, n - nc)])
    t = np.concatenate([ct[k] + 0.08 * r.normal(nc), r.uniform(0, 1, n - nc)])
    p = r.permutation(n)
    res = 1.0 / 64.0
    return Workload("tiny", _pack(x[p], y[p], t[p], (1.0, 1.0, 1.0)), (0.0, 0.0, 0.0),
                    res, res, (64, 64, 64), 3 * res, 3 * res)


def _dengue(seed=2):
    # configs[1]: n=11000; 200 spatial clusters, Zipf(1.2) weights over 256x256;
    # time = 3 seasonal Gaussian bumps over 128 steps; hs=8, ht=5 voxels.
    r = SplitMix64(seed)
    n, K = 11000, 200
    cx, cy = r.uniform(0, 256, K), r.uniform(0, 256, K)
    k = r.categorical(r.zipf_weights(1.2, K), n)
    x = cx[k] + 3.0 * r.normal(n)
    y = cy[k] + 3.0 * r.normal(n)
    bumps = 128.0 * np.array([1 / 6, 1 / 2, 5 / 6])
    b = r.categorical(np.ones(3), n)
    t = bumps[b] + 8.0 * r.normal(n)
    return Workload("dengue", _pack(x, y, t, (256, 256, 128)), (0.0, 0.0, 0.0),
                    1.0, 1.0, (256, 256, 128), 8.0, 5.0)


def _social(seed=3):
    # configs[2]: n=600000; 95% from 50 hotspots (Zipf 1.5, sigma log-uniform
    # in [2,20]) + 5% uniform; 1024x512x256; weekly periodicity; hs=6, ht=4.
    r = SplitMix64(seed)
    n, K = 600000, 50
    nh = int(round(0.95 * n))
    cx, cy = r.uniform(0, 1024, K), r.uniform(0, 512, K)
    sig = np.exp(np.log(2.0) + r.uniform01(K) * (np.log(20.0) - np.log(2.0)))
    k = r.categorical(r.zipf_weights(1.5, K), nh)
    x = np.concatenate([cx[k] + sig[k] * r.normal(nh), r.uniform(0, 1024, n - nh)])
    y = np.concatenate([cy[k] + sig[k] * r.normal(nh), r.uniform(0, 512, n - nh)])
    days = np.arange(256, dtype=np.float64)
    d = r.categorical(1.0 + 0.5 * np.cos(2.0 * np.pi * days / 7.0), n)
    t = d + (1.0 - r.uniform01(n))
    p = r.permutation(n)
    return Workload("social", _pack(x[p], y[p], t[p], (1024, 512, 256)), (0.0, 0.0, 0.0),
                    1.0, 1.0, (1024, 512, 256), 6.0, 4.0)


def _ornith(seed=4):
    # configs[3]: n=5e6 along 20 random 6-vertex polylines; N(0,5^2) jitter in
    # xy; time drifts along each line (t0 + s*D + N(0,5^2)); 2048x1024x365;
    # hs=10, ht=7.
    r = SplitMix64(seed)
    n, L, V = 5_000_000, 20, 6
    vx = r.uniform(0, 2048, L * V).reshape(L, V)
    vy = r.uniform(0, 1024, L * V).reshape(L, V)
    D = r.uniform(90, 270, L)
    t0 = r.uniform(0, 1, L) * (365.0 - D)
    seg = np.hypot(np.diff(vx, axis=1), np.diff(vy, axis=1))      # [L, V-1]
    cum = np.concatenate([np.zeros((L, 1)), np.cumsum(seg, axis=1)], axis=1)
    line = r.categorical(np.ones(L), n)
    s = 1.0 - r.uniform01(n)                                       # [0,1)
    a = s * cum[line, -1]                                          # arc length
    j = np.empty(n, dtype=np.int64)
    for li in range(L):                                            # segment per point
        m = line == li
        j[m] = np.clip(np.searchsorted(cum[li], a[m], side="right") - 1, 0, V - 2)
    segl = np.maximum(seg[line, j], 1e-300)
    f = (a - cum[line, j]) / segl
    px = vx[line, j] + f * (vx[line, j + 1] - vx[line, j])
    py = vy[line, j] + f * (vy[line, j + 1] - vy[line, j])
    x = px + 5.0 * r.normal(n)
    y = py + 5.0 * r.normal(n)
    t = t0[line] + s * D[line] + 5.0 * r.normal(n)
    return Workload("ornith", _pack(x, y, t, (2048, 1024, 365)), (0.0, 0.0, 0.0),
                    1.0, 1.0, (2048, 1024, 365), 10.0, 7.0)


def _stress(seed=5):
    # configs[4]: n=1e6, 50% uniform + 50% from 16 Gaussians sigma=(48,48,32);
    # 1024x1024x512; hs = ht = 32 voxels.
    r = SplitMix64(seed)
    n, K = 1_000_000, 16
    nu = n // 2
    nc = n - nu
    cx, cy, ct = r.uniform(0, 1024, K), r.uniform(0, 1024, K), r.uniform(0, 512, K)
    k = r.categorical(np.ones(K), nc)
    x = np.concatenate([r.uniform(0, 1024, nu), cx[k] + 48.0 * r.normal(nc)])
    y = np.concatenate([r.uniform(0, 1024, nu), cy[k] + 48.0 * r.normal(nc)])
    t = np.concatenate([r.uniform(0, 512, nu), ct[k] + 32.0 * r.normal(nc)])
    p = r.permutation(n)
    return Workload("stress", _pack(x[p], y[p], t[p], (1024, 1024, 512)), (0.0, 0.0, 0.0),
                    1.0, 1.0, (1024, 1024, 512), 32.0, 32.0)


CONFIGS = {"tiny": _tiny, "dengue": _dengue, "social": _social,
           "ornith": _ornith, "stress": _stress}


def make_config(name: str) -> Workload:
    return CONFIGS[name]()


def points_sha256(points: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(points, dtype=np.float32).tobytes()).hexdigest()


def adaptive_bandwidths(w: Workload, lo: float = 0.25) -> np.ndarray:
    """Per-point bandwidths float32 [n, 2] = (hs_i, ht_i) for the adaptive estimator
    (reading R15): a synthetic input recipe, not the
    method.  Abramson's square-root law on a pilot density: rho_i = count of the
    coarse (hs x hs x ht) histogram cell holding point i, lambda_i =
    (rho_i / geometric mean rho)^(-1/2) clamped to [lo, 1], (hs_i, ht_i) =
    lambda_i (hs, ht) -- dense clusters get narrow kernels, sparse background the
    plan's.  Every value is <= the plan's (hs, ht) in FP32 (largest float32 <= h)."""
    p = w.points.astype(np.float64)
    o = np.array(w.origin, np.float64)
    cell = np.array([w.hs, w.hs, w.ht], np.float64)
    nb = np.maximum(np.ceil(np.array(w.G, np.float64) * np.array([w.sres, w.sres, w.tres]) / cell), 1).astype(np.int64)
    idx = np.clip(np.floor((p - o) / cell).astype(np.int64), 0, nb - 1)
    flat = (idx[:, 0] * nb[1] + idx[:, 1]) * nb[2] + idx[:, 2]
    cnt = np.bincount(flat, minlength=int(nb.prod()))[flat].astype(np.float64)
    g = np.exp(np.mean(np.log(cnt)))
    lam = np.clip((cnt / g) ** -0.5, lo, 1.0)

    def cap(h):
        c = np.float32(h)
        return c if float(c) <= h else np.nextafter(c, np.float32(0))
    bw = np.empty((len(p), 2), np.float32)
    bw[:, 0] = np.minimum((lam * w.hs).astype(np.float32), cap(w.hs))
    bw[:, 1] = np.minimum((lam * w.ht).astype(np.float32), cap(w.ht))
    return bw


# The multi-bandwidth sweep of the bench: the plan's bandwidth
# and three narrower ones (the paper's Lb / Hb / VHb instance ladder).
SWEEP_FRACTIONS = (1.0, 0.75, 0.5, 0.25)
