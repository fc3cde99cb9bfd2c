"""The direct x-slab gather (include/stkde.h: stkde_ipc_*; sharded.ShardedSTKDE.export_root_grid /
compute_direct / finish_direct) on one GPU.

Two processes share the device: rank 0 (the root) exports its whole grid as a CUDA IPC handle,
rank 1 maps it, and each rank's tile kernel stores its x-slab straight into the root's grid.
The ranks' kernels never wait on one another (the only synchronisation is a host barrier after
each rank's own stream sync), so two processes on one device exercise the same code as two
GPUs over NVLink, minus the link.  The assembled grid must be bitwise the single-process grid,
with the TMA epilogue and with the plain stores an output on another device takes
(STKDE_PLAIN_STORES forces them)."""
import os
import socket

import numpy as np
import pytest

import stkde_synth as synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, plain, q):
    try:
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        if plain:
            os.environ["STKDE_PLAIN_STORES"] = "1"
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from paper_1705_09366_b200.sharded import ShardedSTKDE
        w = synth.make_config(name)
        pts = torch.from_numpy(w.points).cuda()
        sh = ShardedSTKDE(pts, grid=w.grid_kwargs(), rank=rank, world=world, axis="x")
        full = sh.export_root_grid(root=0)
        if rank == 0:
            full.fill_(float("nan"))                      # every voxel must be written by some rank
        dist.barrier()
        sh.compute_direct()
        got = sh.finish_direct()
        if rank == 0:
            ref = sh.plan.compute(pts)
            torch.cuda.synchronize()
            assert not torch.isnan(got).any()
            assert torch.equal(got, ref), "direct gather differs from the single-process grid"
        sh.close()
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))


@pytest.mark.parametrize("name,plain", [("dengue", 0), ("social", 0), ("social", 1), ("ornith", 0)])
def test_direct_gather_two_processes(name, plain):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, name, plain, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=600) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


def test_ipc_handle_offset():
    # the handle covers the whole allocation; the offset locates the tensor inside it
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1705_09366_b200 as S
    big = torch.empty(1 << 20, dtype=torch.float32, device="cuda")
    h0, off0 = S.ipc_handle(big)
    h1, off1 = S.ipc_handle(big[1000:])
    assert len(h0) == 64 and h0 == h1
    assert off1 - off0 == 4000
    with pytest.raises(ValueError):
        S.ipc_handle(torch.empty(4))
