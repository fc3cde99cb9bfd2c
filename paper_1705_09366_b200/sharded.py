"""Multi-GPU decomposition into slabs (one process per GPU, torch.distributed).

The grid is cut into contiguous, cost-balanced slabs along X (axis "x":
stkde_xslab_partition / stkde_compute_xslab, rows [x0, x1) at multiples of the
16-column tile width -- the default for the tcgen05 engine, whose slab tiles are
the full grid's) or along T (axis "t": stkde_slab_partition / stkde_compute_slab,
the temporal split of PAPER.md:415-433; Bt-aligned cuts, refined to 32 layers by
the tcgen05 engine).  Every rank holds the full point set and computes only its
slab; points that cannot reach the slab are culled on the device, so the halo is
implicit and no reduction is needed: voxel tiles are independent.  There is NO
collective on the data path, and every rank's slab is bitwise equal to the same
block of a single-GPU run.

The optional whole-grid gather to one rank runs inside the C library
(`ShardedSTKDE.init_comm` + `gather`: stkde_plan_comm_init / stkde_gather_xslab /
stkde_gather_slab, NCCL point-to-point over NVLink); `gather_slabs` + `assemble`
are the torch.distributed alternative (any backend, gloo on CPU in the tests).
Neither is part of the timed hot path.

The direct gather (x-slabs; `export_root_grid` + `compute_direct` + `finish_direct`) fuses
the gather into the compute: the root exports its full grid once as a CUDA IPC handle
(stkde_ipc_get_handle, shipped with a torch.distributed object broadcast), every other
rank maps it (stkde_ipc_open) and its tile kernel stores its rows straight into the root's
memory over NVLink / NVSwitch while it computes -- no staging buffer and no collective
after the compute, only a stream sync and a barrier.
"""
from __future__ import annotations

from typing import List, Optional, Sequence

import torch
import torch.distributed as dist

from .stkde import IpcMapping, Plan, ipc_handle, nccl_unique_id


def rank_slab(cuts: Sequence[int], rank: int):
    return int(cuts[rank]), int(cuts[rank + 1])


def exchange_root_handle(rank: int, root: int, export, group=None):
    """Broadcast the root's exported buffer: the root calls export() -> (handle, offset) and
    every rank returns the same (handle, offset) (collective over `group`)."""
    obj = [export() if rank == root else None]
    dist.broadcast_object_list(obj, src=root, group=group)
    handle, offset = obj[0]
    return handle, int(offset)


def direct_row_offset(x0: int, G) -> int:
    """Byte offset of grid row x0 in a float32 [Gx][Gy][Gt] grid (the slab's place in the root's grid)."""
    return int(x0) * int(G[1]) * int(G[2]) * 4


def validate_cuts(cuts: Sequence[int], extent: int, granule: int) -> None:
    """Cuts cover [0, extent), are non-decreasing and multiples of `granule` (except the last)."""
    if cuts[0] != 0 or cuts[-1] != extent:
        raise ValueError("cuts must start at 0 and end at %d: %s" % (extent, list(cuts)))
    for a, b in zip(cuts[:-1], cuts[1:]):
        if b < a:
            raise ValueError("cuts must be non-decreasing: %s" % (list(cuts),))
    for c in cuts[1:-1]:
        if c % granule:
            raise ValueError("interior cuts must be multiples of %d: %s" % (granule, list(cuts)))


class ShardedSTKDE:
    """Per-rank driver: plan on the local GPU, this rank's slab, optional gather."""

    def __init__(self, points: torch.Tensor, *, grid: dict, rank: int, world: int, kernel: int = 0,
                 cuts: Optional[Sequence[int]] = None, axis: Optional[str] = None):
        self.rank, self.world = rank, world
        self.points = points
        self.plan = Plan(max_n=max(int(points.shape[0]), 1), kernel=kernel, device=points.device.index, **grid)
        self.G = self.plan.G
        info = self.plan.info()
        self.Bt = info["Bt"]
        tc = info["engine"] == 2
        self.axis = axis if axis is not None else ("x" if tc else "t")
        if self.axis not in ("x", "t"):
            raise ValueError("axis must be 'x' or 't'")
        # Every rank derives the same cuts from the same points (no collective).
        if self.axis == "x":
            self.cuts = list(cuts) if cuts is not None else self.plan.xslab_partition(points, world)
            validate_cuts(self.cuts, self.G[0], 16)
        else:
            self.cuts = list(cuts) if cuts is not None else self.plan.slab_partition(points, world)
            validate_cuts(self.cuts, self.G[2], 32 if tc else self.Bt)
        self.s0, self.s1 = rank_slab(self.cuts, rank)

    def compute(self, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        """This rank's slab ([x1-x0, Gy, Gt] or [Gx, Gy, t1-t0]), normalised with the global n."""
        n = int(self.points.shape[0])
        if self.axis == "x":
            if out is None:
                out = torch.empty((self.s1 - self.s0, self.G[1], self.G[2]), dtype=torch.float32,
                                  device=self.points.device)
            if self.s1 > self.s0:
                self.plan.compute_xslab(self.points, self.s0, self.s1, n_norm=n, out=out, stream=stream)
            return out
        if out is None:
            out = torch.empty((self.G[0], self.G[1], self.s1 - self.s0), dtype=torch.float32,
                              device=self.points.device)
        if self.s1 > self.s0:
            self.plan.compute_slab(self.points, self.s0, self.s1, n_norm=n, out=out, stream=stream)
        return out

    def contributions(self) -> int:
        """This rank's share of the metric's C (x axis: the whole count on rank 0, 0 elsewhere)."""
        if self.axis == "x":
            return int(self.plan.count_contributions(self.points).item()) if self.rank == 0 else 0
        if self.s1 <= self.s0:
            return 0
        return int(self.plan.count_contributions(self.points, self.s0, self.s1).item())

    def init_comm(self, group=None):
        """Create the library's NCCL communicator for `gather` (rank 0's id shipped over `group`)."""
        uid = [nccl_unique_id() if self.rank == 0 else None]
        dist.broadcast_object_list(uid, src=0, group=group)
        self.plan.comm_init(self.world, self.rank, uid[0])

    def gather(self, slab: torch.Tensor, root: int = 0, full: Optional[torch.Tensor] = None,
               stream=None) -> Optional[torch.Tensor]:
        """The whole grid on `root` (None elsewhere) by the library's NCCL gather; asynchronous."""
        if self.rank == root and full is None:
            full = torch.empty(self.G, dtype=torch.float32, device=self.points.device)
        fn = self.plan.gather_xslab if self.axis == "x" else self.plan.gather_slab
        fn(slab, self.cuts, root, full if self.rank == root else None, stream=stream)
        return full if self.rank == root else None

    # ---- direct gather over peer memory (x-slabs) ----
    def export_root_grid(self, root: int = 0, full: Optional[torch.Tensor] = None, group=None):
        """Collective: the root allocates (or takes) the whole grid and exports it; the other
        ranks map it.  Returns the grid on the root, None elsewhere."""
        if self.axis != "x":
            raise ValueError("the direct gather needs x-slabs (each slab is a contiguous block of rows)")
        self.root = root
        if self.rank == root:
            self.full = full if full is not None else torch.empty(self.G, dtype=torch.float32,
                                                                  device=self.points.device)
        handle, self._root_off = exchange_root_handle(self.rank, root, lambda: ipc_handle(self.full), group)
        if self.rank != root:
            self._peer = IpcMapping(handle, self.points.device.index)
        return self.full if self.rank == root else None

    def compute_direct(self, stream=None) -> None:
        """This rank's slab, stored by the tile kernel straight into the root's grid (asynchronous)."""
        if self.s1 <= self.s0:
            return
        off = direct_row_offset(self.s0, self.G)
        ptr = self.full.data_ptr() + off if self.rank == self.root else self._peer.ptr(self._root_off + off)
        self.plan.compute_xslab_to(self.points, self.s0, self.s1, ptr, n_norm=int(self.points.shape[0]),
                                   stream=stream)

    def finish_direct(self, group=None) -> Optional[torch.Tensor]:
        """Every rank's stores complete (device sync + barrier); the whole grid on the root."""
        torch.cuda.synchronize(self.points.device)
        dist.barrier(group=group)
        return self.full if self.rank == self.root else None

    def close(self):
        peer = getattr(self, "_peer", None)
        if peer is not None:
            peer.close()
            self._peer = None
        self.plan.close()


def gather_slabs(slab: torch.Tensor, cuts: Sequence[int], G, root: int = 0, group=None,
                 axis: str = "t") -> Optional[List[torch.Tensor]]:
    """Point-to-point gather of every rank's slab to `root` (returns the list on root)."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if rank != root:
        if slab.numel():
            dist.send(slab.contiguous(), dst=root, group=group)
        return None
    out = []
    for r in range(world):
        t0, t1 = rank_slab(cuts, r)
        if r == root:
            out.append(slab)
        else:
            shape = (t1 - t0, G[1], G[2]) if axis == "x" else (G[0], G[1], t1 - t0)
            buf = torch.empty(shape, dtype=slab.dtype, device=slab.device)
            if buf.numel():
                dist.recv(buf, src=r, group=group)
            out.append(buf)
    return out


def assemble(slabs: Sequence[torch.Tensor], cuts: Sequence[int], G, axis: str = "t") -> torch.Tensor:
    """Write per-rank slabs ([x1-x0, Gy, Gt] or [Gx, Gy, t1-t0]) into the full grid [Gx, Gy, Gt]."""
    full = torch.empty((G[0], G[1], G[2]), dtype=slabs[0].dtype, device=slabs[0].device)
    for r, s in enumerate(slabs):
        a, b = rank_slab(cuts, r)
        if b > a:
            if axis == "x":
                full[a:b] = s
            else:
                full[:, :, a:b] = s
    return full
