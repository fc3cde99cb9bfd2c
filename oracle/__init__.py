"""FP64 CPU oracle for STKDE (ctypes wrapper over oracle/stkde_oracle.c).

TEST INFRASTRUCTURE ONLY: importable from tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  The product package
(paper_1705_09366_b200/) never imports this module, and this module never
imports the product package.  See stkde_oracle.c for the paper passages each
function follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "stkde_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (OpenMP, -ffp-contract=off).  Returns the .so path."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
                               "-fPIC", "-shared", "-Wall", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Grid(ctypes.Structure):
    _fields_ = [("x0", ctypes.c_double), ("y0", ctypes.c_double), ("t0", ctypes.c_double),
                ("sres", ctypes.c_double), ("tres", ctypes.c_double),
                ("hs", ctypes.c_double), ("ht", ctypes.c_double),
                ("Gx", ctypes.c_int64), ("Gy", ctypes.c_int64), ("Gt", ctypes.c_int64),
                ("kernel", ctypes.c_int32), ("pad_", ctypes.c_int32)]


_lib = None


def _L():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P, I64, I32, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        _lib.oracle_pb.argtypes = [P, I64, P, P, P, P, P, I32]
        _lib.oracle_vb.argtypes = [P, I64, P, P, P, P, P]
        _lib.oracle_vb_voxels.argtypes = [P, I64, P, P, I64, P, P, P, I32]
        _lib.oracle_contributions.argtypes = [P, I64, P, P, I32]
        _lib.oracle_k_s.argtypes = [ctypes.c_int32, D, D]
        _lib.oracle_k_s.restype = D
        _lib.oracle_k_t.argtypes = [ctypes.c_int32, D]
        _lib.oracle_k_t.restype = D
        _lib.oracle_H.argtypes = [D, D]
        _lib.oracle_H.restype = I64
        _lib.oracle_pb_adaptive.argtypes = [P, P, I64, P, P, P, P, P, I32]
        _lib.oracle_vb_adaptive.argtypes = [P, P, I64, P, P, P, P, P]
        _lib.oracle_vb_voxels_adaptive.argtypes = [P, P, I64, P, P, I64, P, P, P, I32]
        _lib.oracle_contributions_adaptive.argtypes = [P, P, I64, P, P, I32]
        for f in (_lib.oracle_pb, _lib.oracle_vb, _lib.oracle_vb_voxels, _lib.oracle_contributions,
                  _lib.oracle_pb_adaptive, _lib.oracle_vb_adaptive, _lib.oracle_vb_voxels_adaptive,
                  _lib.oracle_contributions_adaptive):
            f.restype = I32
    return _lib


def _grid(x0, y0, t0, sres, tres, Gx, Gy, Gt, hs, ht, kernel=0):
    return _Grid(float(x0), float(y0), float(t0), float(sres), float(tres), float(hs), float(ht),
                 int(Gx), int(Gy), int(Gt), int(kernel), 0)


def _pts(points):
    p = np.ascontiguousarray(points, dtype=np.float32).reshape(-1, 3)
    return p, p.ctypes.data


def _ptr(a):
    return None if a is None else a.ctypes.data


def _bw(bw, n):
    b = np.ascontiguousarray(bw, dtype=np.float32).reshape(-1, 2)
    if b.shape[0] != n:
        raise ValueError("bw must be float32 [n][2] = (hs_i, ht_i)")
    return b, b.ctypes.data


def _rc(rc, what):
    if rc == -3:
        raise ValueError("%s: per-point bandwidths must satisfy 0 < hs_i <= hs, 0 < ht_i <= ht" % what)
    if rc != 0:
        raise ValueError("%s failed: %d" % (what, rc))


class OracleResult:
    def __init__(self, vol, slack, amb, contributions):
        self.vol, self.slack, self.amb, self.contributions = vol, slack, amb, contributions


def stkde_pb(points, *, x0, y0, t0, sres, tres, Gx, Gy, Gt, hs, ht, kernel=0,
             with_ambiguity=True, nthreads=0) -> OracleResult:
    """Point-major FP64 density (Alg. 3 structure; bitwise equal to stkde_vb)."""
    p, pp = _pts(points)
    g = _grid(x0, y0, t0, sres, tres, Gx, Gy, Gt, hs, ht, kernel)
    vol = np.empty((Gx, Gy, Gt), dtype=np.float64)
    slack = np.empty_like(vol) if with_ambiguity else None
    amb = np.empty((Gx, Gy, Gt), dtype=np.uint8) if with_ambiguity else None
    C = ctypes.c_int64(0)
    rc = _L().oracle_pb(pp, p.shape[0], ctypes.byref(g), vol.ctypes.data, _ptr(slack), _ptr(amb),
                        ctypes.addressof(C), int(nthreads))
    if rc != 0:
        raise ValueError("oracle_pb failed: %d" % rc)
    return OracleResult(vol, slack, amb, C.value)


def stkde_vb(points, *, x0, y0, t0, sres, tres, Gx, Gy, Gt, hs, ht, kernel=0) -> OracleResult:
    """Alg. 1 (VB) brute force over every voxel and every point (tiny grids only)."""
    p, pp = _pts(points)
    g = _grid(x0, y0, t0, sres, tres, Gx, Gy, Gt, hs, ht, kernel)
    vol = np.empty((Gx, Gy, Gt), dtype=np.float64)
    slack = np.empty_like(vol)
    amb = np.empty((Gx, Gy, Gt), dtype=np.uint8)
    C = ctypes.c_int64(0)
    rc = _L().oracle_vb(pp, p.shape[0], ctypes.byref(g), vol.ctypes.data, slack.ctypes.data,
                        amb.ctypes.data, ctypes.addressof(C))
    if rc != 0:
        raise ValueError("oracle_vb failed: %d" % rc)
    return OracleResult(vol, slack, amb, C.value)


def stkde_vb_voxels(points, voxels, *, x0, y0, t0, sres, tres, Gx, Gy, Gt, hs, ht, kernel=0,
                    nthreads=0):
    """Alg. 1 at the given linear voxel indices (X*Gy+Y)*Gt+T -> (values, slack, amb)."""
    p, pp = _pts(points)
    g = _grid(x0, y0, t0, sres, tres, Gx, Gy, Gt, hs, ht, kernel)
    vox = np.ascontiguousarray(voxels, dtype=np.int64)
    val = np.empty(len(vox), dtype=np.float64)
    slack = np.empty(len(vox), dtype=np.float64)
    amb = np.empty(len(vox), dtype=np.uint8)
    rc = _L().oracle_vb_voxels(pp, p.shape[0], ctypes.byref(g), vox.ctypes.data, len(vox),
                               val.ctypes.data, slack.ctypes.data, amb.ctypes.data, int(nthreads))
    if rc != 0:
        raise ValueError("oracle_vb_voxels failed: %d" % rc)
    return val, slack, amb


def contributions(points, *, x0, y0, t0, sres, tres, Gx, Gy, Gt, hs, ht, kernel=0, nthreads=0) -> int:
    """Exact number of gated (point, voxel) pairs C."""
    p, pp = _pts(points)
    g = _grid(x0, y0, t0, sres, tres, Gx, Gy, Gt, hs, ht, kernel)
    C = ctypes.c_int64(0)
    rc = _L().oracle_contributions(pp, p.shape[0], ctypes.byref(g), ctypes.addressof(C), int(nthreads))
    if rc != 0:
        raise ValueError("oracle_contributions failed: %d" % rc)
    return C.value


def k_s(u, v, kernel=0) -> float:
    return _L().oracle_k_s(int(kernel), float(u), float(v))


def k_t(w, kernel=0) -> float:
    return _L().oracle_k_t(int(kernel), float(w))


def H(h, res) -> int:
    return _L().oracle_H(float(h), float(res))


# ---- adaptive bandwidth (reading R15) ----
# bw = float32 [n][2] = (hs_i, ht_i) in world units, each <= the grid's (hs, ht),
# which then only bound the loops.  f = 1/n sum_i k_s k_t / (hs_i^2 ht_i).

def stkde_pb_adaptive(points, bw, *, x0, y0, t0, sres, tres, Gx, Gy, Gt, hs, ht, kernel=0,
                      with_ambiguity=True, nthreads=0) -> OracleResult:
    """Point-major FP64 adaptive-bandwidth density (bitwise equal to stkde_vb_adaptive)."""
    p, pp = _pts(points)
    b, bp = _bw(bw, p.shape[0])
    g = _grid(x0, y0, t0, sres, tres, Gx, Gy, Gt, hs, ht, kernel)
    vol = np.empty((Gx, Gy, Gt), dtype=np.float64)
    slack = np.empty_like(vol) if with_ambiguity else None
    amb = np.empty((Gx, Gy, Gt), dtype=np.uint8) if with_ambiguity else None
    C = ctypes.c_int64(0)
    _rc(_L().oracle_pb_adaptive(pp, bp, p.shape[0], ctypes.byref(g), vol.ctypes.data, _ptr(slack), _ptr(amb),
                                ctypes.addressof(C), int(nthreads)), "oracle_pb_adaptive")
    return OracleResult(vol, slack, amb, C.value)


def stkde_vb_adaptive(points, bw, *, x0, y0, t0, sres, tres, Gx, Gy, Gt, hs, ht, kernel=0) -> OracleResult:
    """Alg. 1 brute force with per-point bandwidths (tiny grids only)."""
    p, pp = _pts(points)
    b, bp = _bw(bw, p.shape[0])
    g = _grid(x0, y0, t0, sres, tres, Gx, Gy, Gt, hs, ht, kernel)
    vol = np.empty((Gx, Gy, Gt), dtype=np.float64)
    slack = np.empty_like(vol)
    amb = np.empty((Gx, Gy, Gt), dtype=np.uint8)
    C = ctypes.c_int64(0)
    _rc(_L().oracle_vb_adaptive(pp, bp, p.shape[0], ctypes.byref(g), vol.ctypes.data, slack.ctypes.data,
                                amb.ctypes.data, ctypes.addressof(C)), "oracle_vb_adaptive")
    return OracleResult(vol, slack, amb, C.value)


def stkde_vb_voxels_adaptive(points, bw, voxels, *, x0, y0, t0, sres, tres, Gx, Gy, Gt, hs, ht, kernel=0,
                             nthreads=0):
    """Adaptive Alg. 1 at the given linear voxel indices -> (values, slack, amb)."""
    p, pp = _pts(points)
    b, bp = _bw(bw, p.shape[0])
    g = _grid(x0, y0, t0, sres, tres, Gx, Gy, Gt, hs, ht, kernel)
    vox = np.ascontiguousarray(voxels, dtype=np.int64)
    val = np.empty(len(vox), dtype=np.float64)
    slack = np.empty(len(vox), dtype=np.float64)
    amb = np.empty(len(vox), dtype=np.uint8)
    _rc(_L().oracle_vb_voxels_adaptive(pp, bp, p.shape[0], ctypes.byref(g), vox.ctypes.data, len(vox),
                                       val.ctypes.data, slack.ctypes.data, amb.ctypes.data, int(nthreads)),
        "oracle_vb_voxels_adaptive")
    return val, slack, amb


def contributions_adaptive(points, bw, *, x0, y0, t0, sres, tres, Gx, Gy, Gt, hs, ht, kernel=0,
                           nthreads=0) -> int:
    """Exact number of gated (point, voxel) pairs with per-point bandwidths."""
    p, pp = _pts(points)
    b, bp = _bw(bw, p.shape[0])
    g = _grid(x0, y0, t0, sres, tres, Gx, Gy, Gt, hs, ht, kernel)
    C = ctypes.c_int64(0)
    _rc(_L().oracle_contributions_adaptive(pp, bp, p.shape[0], ctypes.byref(g), ctypes.addressof(C),
                                           int(nthreads)), "oracle_contributions_adaptive")
    return C.value
