"""B200-native space-time kernel density estimation (PB-SYM hot path).

Saule et al., "Parallel Space-Time Kernel Density Estimation" (arXiv 1705.09366):
the point-based separable accumulation PB-SYM (Alg. 3) as a gather-form
sm_100a tile kernel behind a C ABI (include/stkde.h).  This package holds the
CUDA sources (csrc/), the in-tree build (build.py), the ctypes binding
(stkde.py) and the time-slab multi-GPU driver (sharded.py).
"""
from .stkde import (KERNEL_CLASSICAL, KERNEL_PRINTED, EXPORTS, LIB_PATH, Plan, StkdeError,  # noqa: F401
                    STKDE_EBANDWIDTH, STKDE_EINVAL, STKDE_ENONFINITE, FLAG_BANDWIDTH, FLAG_NONFINITE,
                    FLAG_WORKLIST, PHASES, STKDE_ENCCL, IpcMapping, compute_sharded, ipc_handle, load_library,
                    nccl_unique_id, slab_cuts,
                    stkde, xslab_cuts)

__all__ = ["Plan", "StkdeError", "stkde", "compute_sharded", "load_library", "slab_cuts", "KERNEL_PRINTED",
           "KERNEL_CLASSICAL", "EXPORTS", "LIB_PATH", "STKDE_EBANDWIDTH", "STKDE_EINVAL", "STKDE_ENONFINITE", "xslab_cuts",
           "FLAG_NONFINITE", "FLAG_WORKLIST", "FLAG_BANDWIDTH", "PHASES", "STKDE_ENCCL", "nccl_unique_id",
           "ipc_handle", "IpcMapping"]
