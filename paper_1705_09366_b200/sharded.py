"""Time-slab multi-GPU decomposition (one process per GPU, torch.distributed).

The grid is cut along T into contiguous, cost-balanced slabs whose
boundaries are multiples of the tile height Bt (stkde_slab_partition).  Every
rank holds the full point set and computes only its slab with
stkde_compute_slab; points whose temporal window misses the slab are culled on
the device, so the halo of PAPER.md:415-433's temporal split is implicit and no
reduction is needed: voxel tiles are independent.  There is NO collective on
the data path.  Because slab boundaries are Bt-aligned, every rank's slab is
bitwise equal to the same layers of a single-GPU run.

`gather_slabs` is the optional whole-grid gather to one rank (NCCL point-to-
point over NVLink on GPUs, gloo on CPU in the tests); `assemble` writes the
slabs into the T-innermost full layout.  Neither is part of the timed hot path.
"""
from __future__ import annotations

from typing import List, Optional, Sequence

import torch
import torch.distributed as dist

from .stkde import Plan


def rank_slab(cuts: Sequence[int], rank: int):
    return int(cuts[rank]), int(cuts[rank + 1])


def validate_cuts(cuts: Sequence[int], Gt: int, Bt: int) -> None:
    """Cuts cover [0, Gt), are non-decreasing and Bt-aligned (except the last)."""
    if cuts[0] != 0 or cuts[-1] != Gt:
        raise ValueError("cuts must start at 0 and end at Gt: %s" % (list(cuts),))
    for a, b in zip(cuts[:-1], cuts[1:]):
        if b < a:
            raise ValueError("cuts must be non-decreasing: %s" % (list(cuts),))
    for c in cuts[1:-1]:
        if c % Bt:
            raise ValueError("interior cuts must be multiples of Bt=%d: %s" % (Bt, list(cuts)))


class ShardedSTKDE:
    """Per-rank driver: plan on the local GPU, this rank's slab, optional gather."""

    def __init__(self, points: torch.Tensor, *, grid: dict, rank: int, world: int, kernel: int = 0,
                 cuts: Optional[Sequence[int]] = None):
        self.rank, self.world = rank, world
        self.points = points
        self.plan = Plan(max_n=max(int(points.shape[0]), 1), kernel=kernel, device=points.device.index, **grid)
        self.G = self.plan.G
        self.Bt = self.plan.info()["Bt"]
        # Every rank derives the same cuts from the same points (no collective).
        self.cuts = list(cuts) if cuts is not None else self.plan.slab_partition(points, world)
        validate_cuts(self.cuts, self.G[2], self.Bt)
        self.t0, self.t1 = rank_slab(self.cuts, rank)

    def compute(self, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        """This rank's slab [Gx, Gy, t1-t0], normalised with the global n."""
        if out is None:
            out = torch.empty((self.G[0], self.G[1], self.t1 - self.t0), dtype=torch.float32,
                              device=self.points.device)
        if self.t1 > self.t0:
            self.plan.compute_slab(self.points, self.t0, self.t1, n_norm=int(self.points.shape[0]), out=out,
                                   stream=stream)
        return out

    def contributions(self) -> int:
        if self.t1 <= self.t0:
            return 0
        return int(self.plan.count_contributions(self.points, self.t0, self.t1).item())

    def close(self):
        self.plan.close()


def gather_slabs(slab: torch.Tensor, cuts: Sequence[int], G, root: int = 0, group=None) -> Optional[List[torch.Tensor]]:
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
            buf = torch.empty((G[0], G[1], t1 - t0), dtype=slab.dtype, device=slab.device)
            if buf.numel():
                dist.recv(buf, src=r, group=group)
            out.append(buf)
    return out


def assemble(slabs: Sequence[torch.Tensor], cuts: Sequence[int], G) -> torch.Tensor:
    """Write per-rank slabs [Gx, Gy, t1-t0] into the full T-innermost grid [Gx, Gy, Gt]."""
    full = torch.empty((G[0], G[1], G[2]), dtype=slabs[0].dtype, device=slabs[0].device)
    for r, s in enumerate(slabs):
        t0, t1 = rank_slab(cuts, r)
        if t1 > t0:
            full[:, :, t0:t1] = s
    return full
