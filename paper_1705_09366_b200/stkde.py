"""Thin ctypes binding over libstkde.so (include/stkde.h).

Argument marshalling only: every step of the density computation runs in the
CUDA kernels of csrc/.  There is no CPU fallback -- if the library or a CUDA
device is missing the calls raise.  PyTorch supplies device memory, streams
and (for the sharded path) process groups.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libstkde.so")

STKDE_OK, STKDE_EINVAL, STKDE_ENOMEM, STKDE_ECUDA, STKDE_ECAPACITY, STKDE_ENONFINITE = 0, -1, -2, -3, -4, -5
STKDE_EBANDWIDTH, STKDE_ENCCL = -6, -7
FLAG_NONFINITE, FLAG_WORKLIST, FLAG_BANDWIDTH = 1, 2, 4
KERNEL_PRINTED, KERNEL_CLASSICAL = 0, 1
# stkde_plan_phase_ms order (STKDE_PHASE_*)
PHASES = ("prep", "sort", "scan", "scatter", "chords", "worklist", "tiles", "gather")

# Exported entry points of include/stkde.h (checked by tests/test_abi.py).
EXPORTS = ("stkde_plan_create", "stkde_plan_destroy", "stkde_compute", "stkde_compute_slab",
           "stkde_slab_partition", "stkde_slab_cuts", "stkde_count_contributions", "stkde_compute_sharded",
           "stkde_plan_check", "stkde_plan_info", "stkde_plan_enable_kernel_timing",
           "stkde_plan_kernel_ms", "stkde_plan_mma_stats", "stkde_plan_check_flags", "stkde_count_contributions_box",
           "stkde_graph_create", "stkde_graph_create_xslab", "stkde_graph_launch", "stkde_graph_destroy",
           "stkde_strerror",
           "stkde_last_error", "stkde_compute_adaptive", "stkde_compute_adaptive_slab",
           "stkde_count_contributions_adaptive", "stkde_compute_sweep", "stkde_compute_xslab",
           "stkde_xslab_partition", "stkde_xslab_cuts", "stkde_compute_adaptive_xslab", "stkde_compute_sharded_x",
           "stkde_compute_f64", "stkde_compute_slab_f64", "stkde_compute_adaptive_slab_f64",
           "stkde_plan_enable_phase_timing", "stkde_plan_phase_ms", "stkde_phase_name",
           "stkde_nccl_unique_id", "stkde_plan_comm_init", "stkde_gather_xslab", "stkde_gather_slab",
           "stkde_ipc_get_handle", "stkde_ipc_open", "stkde_ipc_close")


class StkdeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__("stkde error %d: %s" % (code, msg))
        self.code = code


class PlanInfo(ctypes.Structure):
    _fields_ = [("Bx", ctypes.c_int32), ("By", ctypes.c_int32), ("Bt", ctypes.c_int32),
                ("Hs", ctypes.c_int32), ("Ht", ctypes.c_int32),
                ("ntiles", ctypes.c_int64), ("workspace_bytes", ctypes.c_int64),
                ("last_own_launches", ctypes.c_int32), ("last_cub_calls", ctypes.c_int32),
                ("tile_threads", ctypes.c_int32), ("tile_ctas_per_sm", ctypes.c_int32),
                ("num_sms", ctypes.c_int32), ("chunk_candidates", ctypes.c_int32),
                ("tile_layers_per_thread", ctypes.c_int32), ("engine", ctypes.c_int32)]


_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libstkde.so (raises if it was not built: `python -m paper_1705_09366_b200.build`)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("STKDE_LIB_PATH", path)   # development: an alternative in-tree build
    if not os.path.exists(path):
        raise FileNotFoundError("libstkde.so not built at %s (run python -m paper_1705_09366_b200.build)" % path)
    L = ctypes.CDLL(path)
    P, I64, I32, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
    L.stkde_plan_create.argtypes = [ctypes.POINTER(P), I32, D, D, D, D, D, I64, I64, I64, D, D, I32, I64]
    L.stkde_plan_destroy.argtypes = [P]
    L.stkde_plan_destroy.restype = None
    L.stkde_compute.argtypes = [P, P, I64, P, P]
    L.stkde_compute_slab.argtypes = [P, P, I64, I64, I64, I64, P, P]
    L.stkde_slab_partition.argtypes = [P, P, I64, I32, ctypes.POINTER(I64), P]
    L.stkde_slab_cuts.argtypes = [I64, I64, I64, I32, I32, D, ctypes.POINTER(I64), I32, ctypes.POINTER(I64)]
    L.stkde_count_contributions.argtypes = [P, P, I64, I64, I64, P, P]
    L.stkde_compute_sharded.argtypes = [ctypes.POINTER(P), I32, ctypes.POINTER(P), I64, ctypes.POINTER(P),
                                        ctypes.POINTER(I64), I32, P, ctypes.POINTER(P)]
    L.stkde_plan_check.argtypes = [P]
    L.stkde_plan_info.argtypes = [P, ctypes.POINTER(PlanInfo)]
    L.stkde_plan_enable_kernel_timing.argtypes = [P, I32]
    L.stkde_plan_kernel_ms.argtypes = [P, ctypes.POINTER(D), ctypes.POINTER(I64)]
    L.stkde_plan_mma_stats.argtypes = [P, ctypes.POINTER(I64), ctypes.POINTER(I64)]
    L.stkde_plan_check_flags.argtypes = [P, ctypes.POINTER(ctypes.c_uint32)]
    L.stkde_count_contributions_box.argtypes = [P, P, I64, I64, I64, I64, I64, P, P]
    L.stkde_graph_create.argtypes = [P, P, I64, I64, I64, I64, P, ctypes.POINTER(P)]
    L.stkde_graph_create_xslab.argtypes = [P, P, I64, I64, I64, I64, P, ctypes.POINTER(P)]
    L.stkde_graph_launch.argtypes = [P, P]
    L.stkde_graph_destroy.argtypes = [P]
    L.stkde_graph_destroy.restype = None
    # development diagnostics: exported only by a -DSTKDE_TC_DIAG=1 build (csrc/stkde_diag.h)
    DIAG = ("stkde_plan_tc_profile", "stkde_plan_debug_progress")
    if hasattr(L, DIAG[0]):
        L.stkde_plan_tc_profile.argtypes = [P, ctypes.POINTER(ctypes.c_uint64)]
        L.stkde_plan_debug_progress.argtypes = [P, P]
    L.stkde_compute_adaptive.argtypes = [P, P, P, I64, P, P]
    L.stkde_compute_adaptive_slab.argtypes = [P, P, P, I64, I64, I64, I64, P, P]
    L.stkde_count_contributions_adaptive.argtypes = [P, P, P, I64, I64, I64, P, P]
    L.stkde_compute_sweep.argtypes = [P, P, I64, I32, ctypes.POINTER(D), ctypes.POINTER(D), ctypes.POINTER(P), P]
    L.stkde_compute_xslab.argtypes = [P, P, I64, I64, I64, I64, P, P]
    L.stkde_compute_adaptive_xslab.argtypes = [P, P, P, I64, I64, I64, I64, P, P]
    L.stkde_compute_sharded_x.argtypes = [ctypes.POINTER(P), I32, ctypes.POINTER(P), I64, ctypes.POINTER(P),
                                          ctypes.POINTER(I64), I32, P, ctypes.POINTER(P)]
    L.stkde_xslab_partition.argtypes = [P, P, I64, I32, ctypes.POINTER(I64), P]
    L.stkde_xslab_cuts.argtypes = [I64, I64, I64, D, D, ctypes.POINTER(I64), I32, ctypes.POINTER(I64)]
    L.stkde_compute_f64.argtypes = [P, P, I64, P, P]
    L.stkde_compute_slab_f64.argtypes = [P, P, I64, I64, I64, I64, P, P]
    L.stkde_compute_adaptive_slab_f64.argtypes = [P, P, P, I64, I64, I64, I64, P, P]
    L.stkde_plan_enable_phase_timing.argtypes = [P, I32]
    L.stkde_plan_phase_ms.argtypes = [P, ctypes.POINTER(D), ctypes.POINTER(I64)]
    L.stkde_phase_name.argtypes = [I32]
    L.stkde_phase_name.restype = ctypes.c_char_p
    L.stkde_nccl_unique_id.argtypes = [P]
    L.stkde_plan_comm_init.argtypes = [P, I32, I32, P]
    L.stkde_gather_xslab.argtypes = [P, P, ctypes.POINTER(I64), I32, P, P]
    L.stkde_gather_slab.argtypes = [P, P, ctypes.POINTER(I64), I32, P, P]
    L.stkde_ipc_get_handle.argtypes = [P, P, ctypes.POINTER(I64)]
    L.stkde_ipc_open.argtypes = [I32, P, ctypes.POINTER(P)]
    L.stkde_ipc_close.argtypes = [P]
    L.stkde_strerror.argtypes = [I32]
    L.stkde_strerror.restype = ctypes.c_char_p
    L.stkde_last_error.argtypes = []
    L.stkde_last_error.restype = ctypes.c_char_p
    for name in ("stkde_plan_create", "stkde_compute", "stkde_compute_slab", "stkde_slab_partition", "stkde_slab_cuts",
                 "stkde_count_contributions", "stkde_compute_sharded", "stkde_plan_check",
                 "stkde_plan_info", "stkde_plan_enable_kernel_timing", "stkde_plan_kernel_ms",
                 "stkde_plan_mma_stats", "stkde_plan_check_flags", "stkde_count_contributions_box",
                 "stkde_graph_create", "stkde_graph_create_xslab", "stkde_graph_launch", "stkde_compute_adaptive", "stkde_compute_adaptive_slab", "stkde_count_contributions_adaptive",
                 "stkde_compute_sweep", "stkde_compute_xslab", "stkde_xslab_partition", "stkde_xslab_cuts",
                 "stkde_compute_adaptive_xslab", "stkde_compute_sharded_x", "stkde_compute_f64",
                 "stkde_compute_slab_f64", "stkde_compute_adaptive_slab_f64", "stkde_plan_enable_phase_timing",
                 "stkde_plan_phase_ms", "stkde_nccl_unique_id", "stkde_plan_comm_init", "stkde_gather_xslab",
                 "stkde_gather_slab", "stkde_ipc_get_handle", "stkde_ipc_open", "stkde_ipc_close") + (
                     DIAG if hasattr(L, DIAG[0]) else ()):
        getattr(L, name).restype = I32
    _lib = L
    return L


def _check(rc: int):
    if rc != STKDE_OK:
        L = load_library()
        raise StkdeError(rc, L.stkde_last_error().decode() or L.stkde_strerror(rc).decode())
    return rc


def _stream_ptr(stream: Optional[torch.cuda.Stream], device) -> int:
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return int(s.cuda_stream)


def _points_arg(points: torch.Tensor, device: torch.device) -> torch.Tensor:
    if not isinstance(points, torch.Tensor) or points.device != device:
        raise ValueError("points must be a CUDA tensor on %s" % device)
    if points.dtype != torch.float32 or points.dim() != 2 or points.shape[1] != 3:
        raise ValueError("points must be float32 [n, 3] (x, y, t)")
    return points.contiguous()


def _bw_arg(bw: torch.Tensor, device: torch.device, n: int) -> torch.Tensor:
    if not isinstance(bw, torch.Tensor) or bw.device != device:
        raise ValueError("bw must be a CUDA tensor on %s" % device)
    if bw.dtype != torch.float32 or bw.dim() != 2 or bw.shape[1] != 2 or bw.shape[0] != n:
        raise ValueError("bw must be float32 [n, 2] (hs_i, ht_i)")
    return bw.contiguous()


class Plan:
    """A density plan on one device (stkde_plan_create); owns the device workspace."""

    def __init__(self, *, x0, y0, t0, sres, tres, Gx, Gy, Gt, hs, ht, max_n: int,
                 kernel: int = KERNEL_PRINTED, device=None):
        L = load_library()
        if device is None:
            device = torch.cuda.current_device()
        self.device = torch.device("cuda", device if isinstance(device, int) else torch.device(device).index)
        self.G = (int(Gx), int(Gy), int(Gt))
        self.grid = dict(x0=float(x0), y0=float(y0), t0=float(t0), sres=float(sres), tres=float(tres),
                         Gx=int(Gx), Gy=int(Gy), Gt=int(Gt), hs=float(hs), ht=float(ht))
        self.kernel = int(kernel)
        self.max_n = int(max_n)
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _check(L.stkde_plan_create(ctypes.byref(h), self.device.index, float(x0), float(y0), float(t0),
                                       float(sres), float(tres), int(Gx), int(Gy), int(Gt), float(hs), float(ht),
                                       int(kernel), int(max_n)))
        self._h = h

    # -- lifecycle --
    def close(self):
        if getattr(self, "_h", None):
            load_library().stkde_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    # -- compute --
    def compute(self, points: torch.Tensor, out: Optional[torch.Tensor] = None,
                stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """Full grid [Gx, Gy, Gt] float32 (fully overwritten)."""
        pts = _points_arg(points, self.device)
        if out is None:
            out = torch.empty(self.G, dtype=torch.float32, device=self.device)
        self._check_out(out, self.G[2])
        _check(load_library().stkde_compute(self._h, pts.data_ptr(), pts.shape[0], out.data_ptr(),
                                             _stream_ptr(stream, self.device)))
        return out

    def compute_slab(self, points: torch.Tensor, t_begin: int, t_end: int, n_norm: Optional[int] = None,
                     out: Optional[torch.Tensor] = None, stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """Time slab [t_begin, t_end): [Gx, Gy, t_end - t_begin] float32, normalised with n_norm."""
        pts = _points_arg(points, self.device)
        ts = int(t_end) - int(t_begin)
        if out is None:
            out = torch.empty((self.G[0], self.G[1], max(ts, 0)), dtype=torch.float32, device=self.device)
        self._check_out(out, ts)
        nn = pts.shape[0] if n_norm is None else int(n_norm)
        _check(load_library().stkde_compute_slab(self._h, pts.data_ptr(), pts.shape[0], nn, int(t_begin),
                                                 int(t_end), out.data_ptr(), _stream_ptr(stream, self.device)))
        return out

    def graph(self, points: torch.Tensor, out: Optional[torch.Tensor] = None, t_begin: int = 0,
              t_end: Optional[int] = None, n_norm: Optional[int] = None) -> "Graph":
        """Capture one compute_slab call (default: the full grid) as a CUDA graph (stkde_graph_create):
        Graph.launch() replays the whole pass with one launch, reading `points` and writing `out`
        as they are at launch time."""
        pts = _points_arg(points, self.device)
        t1 = self.G[2] if t_end is None else int(t_end)
        ts = t1 - int(t_begin)
        if out is None:
            out = torch.empty((self.G[0], self.G[1], max(ts, 0)), dtype=torch.float32, device=self.device)
        self._check_out(out, ts)
        nn = pts.shape[0] if n_norm is None else int(n_norm)
        h = ctypes.c_void_p()
        _check(load_library().stkde_graph_create(self._h, pts.data_ptr(), pts.shape[0], nn, int(t_begin), t1,
                                                 out.data_ptr(), ctypes.byref(h)))
        return Graph(h, self, pts, out)

    def graph_xslab(self, points: torch.Tensor, x_begin: int, x_end: int, n_norm: Optional[int] = None,
                    out: Optional[torch.Tensor] = None) -> "Graph":
        """Capture one compute_xslab call as a CUDA graph (stkde_graph_create_xslab)."""
        pts = _points_arg(points, self.device)
        if out is None:
            out = torch.empty((int(x_end) - int(x_begin), self.G[1], self.G[2]), dtype=torch.float32,
                              device=self.device)
        nn = pts.shape[0] if n_norm is None else int(n_norm)
        h = ctypes.c_void_p()
        _check(load_library().stkde_graph_create_xslab(self._h, pts.data_ptr(), pts.shape[0], nn, int(x_begin),
                                                       int(x_end), out.data_ptr(), ctypes.byref(h)))
        return Graph(h, self, pts, out)

    # -- adaptive bandwidth (include/stkde.h; reading R15) --
    def compute_adaptive(self, points: torch.Tensor, bw: torch.Tensor, out: Optional[torch.Tensor] = None,
                         stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """Full grid with per-point bandwidths bw = float32 [n, 2] (hs_i, ht_i) <= the plan's."""
        pts = _points_arg(points, self.device)
        b = _bw_arg(bw, self.device, pts.shape[0])
        if out is None:
            out = torch.empty(self.G, dtype=torch.float32, device=self.device)
        self._check_out(out, self.G[2])
        _check(load_library().stkde_compute_adaptive(self._h, pts.data_ptr(), b.data_ptr(), pts.shape[0],
                                                      out.data_ptr(), _stream_ptr(stream, self.device)))
        return out

    def compute_adaptive_slab(self, points: torch.Tensor, bw: torch.Tensor, t_begin: int, t_end: int,
                              n_norm: Optional[int] = None, out: Optional[torch.Tensor] = None,
                              stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        pts = _points_arg(points, self.device)
        b = _bw_arg(bw, self.device, pts.shape[0])
        ts = int(t_end) - int(t_begin)
        if out is None:
            out = torch.empty((self.G[0], self.G[1], max(ts, 0)), dtype=torch.float32, device=self.device)
        self._check_out(out, ts)
        nn = pts.shape[0] if n_norm is None else int(n_norm)
        _check(load_library().stkde_compute_adaptive_slab(self._h, pts.data_ptr(), b.data_ptr(), pts.shape[0], nn,
                                                           int(t_begin), int(t_end), out.data_ptr(),
                                                           _stream_ptr(stream, self.device)))
        return out

    # -- FP64 output (include/stkde.h) --
    def compute_f64(self, points: torch.Tensor, t_begin: int = 0, t_end: Optional[int] = None,
                    n_norm: Optional[int] = None, bw: Optional[torch.Tensor] = None,
                    out: Optional[torch.Tensor] = None, stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """float64 [Gx, Gy, t_end - t_begin]: every term in FP64 with Alg. 1's operation
        sequence; bw = per-point (hs_i, ht_i) for the adaptive estimator (None: fixed)."""
        pts = _points_arg(points, self.device)
        t_end = self.G[2] if t_end is None else int(t_end)
        ts = t_end - int(t_begin)
        if out is None:
            out = torch.empty((self.G[0], self.G[1], max(ts, 0)), dtype=torch.float64, device=self.device)
        self._check_out(out, ts, torch.float64)
        nn = pts.shape[0] if n_norm is None else int(n_norm)
        L, st = load_library(), _stream_ptr(stream, self.device)
        if bw is None:
            _check(L.stkde_compute_slab_f64(self._h, pts.data_ptr(), pts.shape[0], nn, int(t_begin), t_end,
                                            out.data_ptr(), st))
        else:
            b = _bw_arg(bw, self.device, pts.shape[0])
            _check(L.stkde_compute_adaptive_slab_f64(self._h, pts.data_ptr(), b.data_ptr(), pts.shape[0], nn,
                                                     int(t_begin), t_end, out.data_ptr(), st))
        return out

    def count_contributions_adaptive(self, points: torch.Tensor, bw: torch.Tensor, t_begin: int = 0,
                                     t_end: Optional[int] = None,
                                     stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        pts = _points_arg(points, self.device)
        b = _bw_arg(bw, self.device, pts.shape[0])
        out = torch.empty(1, dtype=torch.int64, device=self.device)
        _check(load_library().stkde_count_contributions_adaptive(
            self._h, pts.data_ptr(), b.data_ptr(), pts.shape[0], int(t_begin),
            int(self.G[2] if t_end is None else t_end), out.data_ptr(), _stream_ptr(stream, self.device)))
        return out

    # -- x-slabs (include/stkde.h) --
    def compute_xslab(self, points: torch.Tensor, x_begin: int, x_end: int, n_norm: Optional[int] = None,
                      out: Optional[torch.Tensor] = None, stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """Grid rows [x_begin, x_end): [x_end - x_begin, Gy, Gt] float32 (bitwise those rows of compute)."""
        pts = _points_arg(points, self.device)
        shape = (int(x_end) - int(x_begin), self.G[1], self.G[2])
        if out is None:
            out = torch.empty(shape, dtype=torch.float32, device=self.device)
        if out.device != self.device or out.dtype != torch.float32 or not out.is_contiguous() or tuple(out.shape) != shape:
            raise ValueError("out must be a contiguous float32 CUDA tensor of shape %s" % (shape,))
        nn = pts.shape[0] if n_norm is None else int(n_norm)
        _check(load_library().stkde_compute_xslab(self._h, pts.data_ptr(), pts.shape[0], nn, int(x_begin), int(x_end),
                                                  out.data_ptr(), _stream_ptr(stream, self.device)))
        return out

    def compute_xslab_to(self, points: torch.Tensor, x_begin: int, x_end: int, out_ptr: int,
                         n_norm: Optional[int] = None, stream: Optional[torch.cuda.Stream] = None) -> None:
        """Rows [x_begin, x_end) written at device address out_ptr (float32 [x_end - x_begin][Gy][Gt],
        e.g. the rows of the root's grid mapped with IpcMapping: the direct gather)."""
        pts = _points_arg(points, self.device)
        nn = pts.shape[0] if n_norm is None else int(n_norm)
        _check(load_library().stkde_compute_xslab(self._h, pts.data_ptr(), pts.shape[0], nn, int(x_begin), int(x_end),
                                                  ctypes.c_void_p(int(out_ptr)), _stream_ptr(stream, self.device)))

    def compute_adaptive_xslab(self, points: torch.Tensor, bw: torch.Tensor, x_begin: int, x_end: int,
                               n_norm: Optional[int] = None, out: Optional[torch.Tensor] = None,
                               stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """Adaptive-bandwidth grid rows [x_begin, x_end): [x_end - x_begin, Gy, Gt] float32."""
        pts = _points_arg(points, self.device)
        b = _bw_arg(bw, self.device, pts.shape[0])
        shape = (int(x_end) - int(x_begin), self.G[1], self.G[2])
        if out is None:
            out = torch.empty(shape, dtype=torch.float32, device=self.device)
        if out.device != self.device or out.dtype != torch.float32 or not out.is_contiguous() or tuple(out.shape) != shape:
            raise ValueError("out must be a contiguous float32 CUDA tensor of shape %s" % (shape,))
        nn = pts.shape[0] if n_norm is None else int(n_norm)
        _check(load_library().stkde_compute_adaptive_xslab(self._h, pts.data_ptr(), b.data_ptr(), pts.shape[0], nn,
                                                           int(x_begin), int(x_end), out.data_ptr(),
                                                           _stream_ptr(stream, self.device)))
        return out

    def xslab_partition(self, points: torch.Tensor, nparts: int,
                        stream: Optional[torch.cuda.Stream] = None) -> list:
        pts = _points_arg(points, self.device)
        cuts = (ctypes.c_int64 * (nparts + 1))()
        _check(load_library().stkde_xslab_partition(self._h, pts.data_ptr(), pts.shape[0], int(nparts), cuts,
                                                    _stream_ptr(stream, self.device)))
        return [int(c) for c in cuts]

    # -- multi-bandwidth sweep (include/stkde.h) --
    def compute_sweep(self, points: torch.Tensor, hs: Sequence[float], ht: Sequence[float],
                      outs: Optional[Sequence[torch.Tensor]] = None,
                      stream: Optional[torch.cuda.Stream] = None) -> list:
        """One binning, len(hs) grids: grid k at bandwidths (hs[k], ht[k]) <= the plan's."""
        pts = _points_arg(points, self.device)
        k = len(hs)
        if len(ht) != k or k < 1:
            raise ValueError("hs and ht must be equally long, non-empty")
        if outs is None:
            outs = [torch.empty(self.G, dtype=torch.float32, device=self.device) for _ in range(k)]
        for o in outs:
            self._check_out(o, self.G[2])
        H = (ctypes.c_double * k)(*[float(v) for v in hs])
        T = (ctypes.c_double * k)(*[float(v) for v in ht])
        ptrs = (ctypes.c_void_p * k)(*[o.data_ptr() for o in outs])
        _check(load_library().stkde_compute_sweep(self._h, pts.data_ptr(), pts.shape[0], k, H, T, ptrs,
                                                  _stream_ptr(stream, self.device)))
        return list(outs)

    def _check_out(self, out, ts, dtype=torch.float32):
        if out.device != self.device or out.dtype != dtype or not out.is_contiguous() \
                or tuple(out.shape) != (self.G[0], self.G[1], ts):
            raise ValueError("out must be a contiguous %s CUDA tensor of shape %s"
                             % (dtype, (self.G[0], self.G[1], ts)))

    def slab_partition(self, points: torch.Tensor, nparts: int,
                       stream: Optional[torch.cuda.Stream] = None) -> list:
        pts = _points_arg(points, self.device)
        cuts = (ctypes.c_int64 * (nparts + 1))()
        _check(load_library().stkde_slab_partition(self._h, pts.data_ptr(), pts.shape[0], int(nparts), cuts,
                                                   _stream_ptr(stream, self.device)))
        return [int(c) for c in cuts]

    def count_contributions(self, points: torch.Tensor, t_begin: int = 0, t_end: Optional[int] = None,
                            stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """Exact gated (point, voxel) pair count C as a 1-element int64 device tensor (async)."""
        pts = _points_arg(points, self.device)
        out = torch.empty(1, dtype=torch.int64, device=self.device)
        _check(load_library().stkde_count_contributions(
            self._h, pts.data_ptr(), pts.shape[0], int(t_begin), int(self.G[2] if t_end is None else t_end),
            out.data_ptr(), _stream_ptr(stream, self.device)))
        return out

    def count_contributions_box(self, points: torch.Tensor, x_begin: int, x_end: int, t_begin: int = 0,
                                t_end: Optional[int] = None,
                                stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """Exact C restricted to rows [x_begin, x_end) and layers [t_begin, t_end) (async)."""
        pts = _points_arg(points, self.device)
        out = torch.empty(1, dtype=torch.int64, device=self.device)
        _check(load_library().stkde_count_contributions_box(
            self._h, pts.data_ptr(), pts.shape[0], int(x_begin), int(x_end), int(t_begin),
            int(self.G[2] if t_end is None else t_end), out.data_ptr(), _stream_ptr(stream, self.device)))
        return out

    # -- diagnostics --
    def check(self):
        _check(load_library().stkde_plan_check(self._h))

    def check_flags(self) -> int:
        """Every condition raised since the last check (STKDE_FLAG_* bits), then cleared."""
        f = ctypes.c_uint32(0)
        _check(load_library().stkde_plan_check_flags(self._h, ctypes.byref(f)))
        return int(f.value)

    def info(self) -> dict:
        i = PlanInfo()
        _check(load_library().stkde_plan_info(self._h, ctypes.byref(i)))
        return {f: getattr(i, f) for f, _ in PlanInfo._fields_}

    def enable_kernel_timing(self, on: bool = True):
        _check(load_library().stkde_plan_enable_kernel_timing(self._h, 1 if on else 0))

    def kernel_ms(self):
        ms, k = ctypes.c_double(0), ctypes.c_int64(0)
        _check(load_library().stkde_plan_kernel_ms(self._h, ctypes.byref(ms), ctypes.byref(k)))
        return ms.value, k.value

    def enable_phase_timing(self, on: bool = True):
        """CUDA events at every phase end of subsequent calls (stkde_plan_enable_phase_timing)."""
        _check(load_library().stkde_plan_enable_phase_timing(self._h, 1 if on else 0))

    def phase_ms(self):
        """({phase: summed ms since enable}, timed calls) -- synchronises on the last event."""
        ms = (ctypes.c_double * len(PHASES))()
        k = ctypes.c_int64(0)
        _check(load_library().stkde_plan_phase_ms(self._h, ms, ctypes.byref(k)))
        return dict(zip(PHASES, list(ms))), k.value

    # -- NCCL gather of per-rank slabs (one process per GPU) --
    def comm_init(self, nranks: int, rank: int, uid: bytes):
        """Create the plan's NCCL communicator (collective; uid from nccl_unique_id() on rank 0)."""
        if len(uid) != 128:
            raise ValueError("the NCCL unique id is 128 bytes")
        buf = ctypes.create_string_buffer(uid, 128)
        _check(load_library().stkde_plan_comm_init(self._h, int(nranks), int(rank), buf))

    def _gather(self, fn, slab, cuts, root, full, stream):
        if slab.dtype != torch.float32 or not slab.is_contiguous() or slab.device != self.device:
            raise ValueError("slab must be a contiguous float32 tensor on the plan's device")
        if full is not None and (full.dtype != torch.float32 or not full.is_contiguous()
                                 or full.device != self.device or tuple(full.shape) != self.G):
            raise ValueError("full must be a contiguous float32 (Gx, Gy, Gt) tensor on the plan's device")
        c = (ctypes.c_int64 * len(cuts))(*[int(x) for x in cuts])
        _check(fn(self._h, ctypes.c_void_p(slab.data_ptr()), c, int(root),
                  ctypes.c_void_p(full.data_ptr()) if full is not None else None, _stream_ptr(stream, self.device)))
        return full

    def gather_xslab(self, slab: torch.Tensor, cuts: Sequence[int], root: int = 0,
                     full: Optional[torch.Tensor] = None, stream=None):
        """NCCL gather of every rank's x-slab into `full` on `root` (stkde_gather_xslab)."""
        return self._gather(load_library().stkde_gather_xslab, slab, cuts, root, full, stream)

    def gather_slab(self, slab: torch.Tensor, cuts: Sequence[int], root: int = 0,
                    full: Optional[torch.Tensor] = None, stream=None):
        """NCCL gather of every rank's time slab into `full` on `root` (stkde_gather_slab)."""
        return self._gather(load_library().stkde_gather_slab, slab, cuts, root, full, stream)

    def tc_profile(self):
        """32 u64 phase counters of the tcgen05 kernel (STKDE_TC_PROF=1 at plan creation), reset on read."""
        buf = (ctypes.c_uint64 * 32)()
        _check(load_library().stkde_plan_tc_profile(self._h, buf))
        return list(buf)

    def debug_progress(self, ptr: int):
        """Development aid: device-accessible uint32[num_sms * 32] progress buffer (0 = off)."""
        _check(load_library().stkde_plan_debug_progress(self._h, ctypes.c_void_p(ptr) if ptr else None))

    def mma_stats(self):
        """(sum of MMA widths N, k-blocks) issued by the tcgen05 engine since the last call."""
        c, k = ctypes.c_int64(0), ctypes.c_int64(0)
        _check(load_library().stkde_plan_mma_stats(self._h, ctypes.byref(c), ctypes.byref(k)))
        return c.value, k.value


class Graph:
    """A captured compute call (stkde_graph_*); keeps its plan and buffers alive."""

    def __init__(self, h, plan, points, out):
        self._h, self.plan, self.points, self.out = h, plan, points, out

    def launch(self, stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        _check(load_library().stkde_graph_launch(self._h, _stream_ptr(stream, self.plan.device)))
        return self.out

    def close(self):
        if self._h:
            load_library().stkde_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def compute_sharded(plans: Sequence[Plan], points: Sequence[torch.Tensor], slabs: Optional[Sequence[torch.Tensor]],
                    cuts: Optional[Sequence[int]] = None, root: int = -1,
                    full: Optional[torch.Tensor] = None, streams=None, axis: str = "t") -> list:
    """Single-process multi-device driver (stkde_compute_sharded, or stkde_compute_sharded_x for
    axis="x": slabs[d] = rows [cuts[d], cuts[d+1]) as [rows, Gy, Gt]); returns the cuts used."""
    L = load_library()
    nd = len(plans)
    P = ctypes.c_void_p
    hp = (P * nd)(*[p.handle.value for p in plans])
    pts = [_points_arg(x, p.device) for x, p in zip(points, plans)]
    hpts = (P * nd)(*[x.data_ptr() for x in pts])
    # slabs=None with axis="x" and a full grid: the fused gather (stores straight into `full`)
    hsl = None if slabs is None else (P * nd)(*[s.data_ptr() for s in slabs])
    hc = (ctypes.c_int64 * (nd + 1))(*([-1] * (nd + 1) if cuts is None else [int(c) for c in cuts]))
    if streams is None:
        streams = [torch.cuda.current_stream(p.device) for p in plans]
    hs = (P * nd)(*[int(s.cuda_stream) for s in streams])
    fn = L.stkde_compute_sharded_x if axis == "x" else L.stkde_compute_sharded
    _check(fn(hp, nd, hpts, pts[0].shape[0], hsl, hc, int(root), None if full is None else full.data_ptr(), hs))
    return [int(c) for c in hc]


def ipc_handle(t: torch.Tensor):
    """(64-byte CUDA IPC handle of the allocation holding t, t's byte offset in it) -- export a
    device buffer (the root's grid) to the other ranks' processes (stkde_ipc_get_handle)."""
    if not t.is_cuda:
        raise ValueError("ipc_handle needs a CUDA tensor")
    buf = ctypes.create_string_buffer(64)
    off = ctypes.c_int64(0)
    _check(load_library().stkde_ipc_get_handle(ctypes.c_void_p(t.data_ptr()), buf, ctypes.byref(off)))
    return buf.raw, off.value


class IpcMapping:
    """Another process's device allocation mapped into this one (stkde_ipc_open); `ptr(offset)`
    is a device address for the library's pointer-taking calls.  close() unmaps it."""

    def __init__(self, handle: bytes, device: int):
        if len(handle) != 64:
            raise ValueError("a CUDA IPC handle is 64 bytes")
        base = ctypes.c_void_p(0)
        _check(load_library().stkde_ipc_open(int(device), ctypes.create_string_buffer(handle, 64), ctypes.byref(base)))
        self.base = base.value
        self.device = int(device)

    def ptr(self, offset: int = 0) -> int:
        if self.base is None:
            raise ValueError("IPC mapping is closed")
        return self.base + int(offset)

    def close(self):
        if self.base is not None:
            _check(load_library().stkde_ipc_close(ctypes.c_void_p(self.base)))
            self.base = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def nccl_unique_id() -> bytes:
    """A fresh 128-byte NCCL unique id (rank 0; ship it to the other ranks out of band)."""
    buf = ctypes.create_string_buffer(128)
    _check(load_library().stkde_nccl_unique_id(buf))
    return buf.raw


def slab_cuts(G, Bt: int, Ht: int, rs: float, hist_T, nparts: int) -> list:
    """Host-only cost-balanced Bt-aligned cuts from a layer histogram (stkde_slab_cuts)."""
    L = load_library()
    Gt = int(G[2])
    h = (ctypes.c_int64 * Gt)(*[int(v) for v in hist_T])
    cuts = (ctypes.c_int64 * (nparts + 1))()
    _check(L.stkde_slab_cuts(int(G[0]), int(G[1]), Gt, int(Bt), int(Ht), float(rs), h, int(nparts), cuts))
    return [int(c) for c in cuts]


def stkde(points: torch.Tensor, *, x0, y0, t0, sres, tres, Gx, Gy, Gt, hs, ht,
          kernel: int = KERNEL_PRINTED) -> torch.Tensor:
    """One-shot convenience: plan, compute, release."""
    with Plan(x0=x0, y0=y0, t0=t0, sres=sres, tres=tres, Gx=Gx, Gy=Gy, Gt=Gt, hs=hs, ht=ht,
              max_n=max(int(points.shape[0]), 1), kernel=kernel, device=points.device.index) as p:
        out = p.compute(points)
        torch.cuda.current_stream(points.device).synchronize()
        return out


def xslab_cuts(G, rs: float, rt: float, hist_X, nparts: int) -> list:
    """Host-only cost-balanced x cuts (stkde_xslab_cuts): multiples of 16, [0 .. Gx]."""
    L = load_library()
    h = (ctypes.c_int64 * len(hist_X))(*[int(v) for v in hist_X])
    cuts = (ctypes.c_int64 * (nparts + 1))()
    _check(L.stkde_xslab_cuts(int(G[0]), int(G[1]), int(G[2]), float(rs), float(rt), h, int(nparts), cuts))
    return [int(c) for c in cuts]
