"""Host logic of the multi-GPU time-slab path on CPU: the cut computation (C ABI,
host-only call), and a world_size-2 gloo run of cut agreement + slab gather +
assembly against the FP64 oracle's full grid (the oracle stands in for each
rank's device slab; no GPU needed)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import stkde_synth as synth


@pytest.fixture(scope="module")
def S():
    from paper_1705_09366_b200 import build
    build.build()
    import paper_1705_09366_b200 as S
    return S


def hist_T(points, g):
    # test-side layer histogram of T_i = floor((t - t0)/tres), clamped into [0, Gt)
    T = np.floor((points[:, 2].astype(np.float64) - g["t0"]) / g["tres"]).astype(np.int64)
    return np.bincount(np.clip(T, 0, g["Gt"] - 1), minlength=g["Gt"])


@pytest.mark.parametrize("name", ["dengue", "social", "stress"])
@pytest.mark.parametrize("nparts", [1, 2, 3, 8])
def test_cut_properties(S, name, nparts):
    w = synth.make_config(name)
    g = w.grid_kwargs()
    Bt = 64 if w.ht / w.tres >= 16 else (32 if w.ht / w.tres >= 6 else 16)
    h = hist_T(w.points, g)
    cuts = S.slab_cuts(w.G, Bt, int(np.ceil(w.ht / w.tres)), w.hs / w.sres, h, nparts)
    from paper_1705_09366_b200.sharded import validate_cuts
    validate_cuts(cuts, w.G[2], Bt)
    assert len(cuts) == nparts + 1
    nblk = -(-w.G[2] // Bt)
    if nparts <= nblk:
        assert all(b > a for a, b in zip(cuts[:-1], cuts[1:])), cuts   # no empty slab


def test_cuts_balance_skewed(S):
    # compute-dominated, all points in the first quarter of the layers: the
    # balanced cut is far from the equal cut
    Gt, Bt = 512, 16
    h = np.zeros(Gt, np.int64)
    h[:128] = 1000000
    cuts = S.slab_cuts((1024, 1024, Gt), Bt, 8, 8.0, h, 4)
    assert cuts[1] < 128 and cuts[2] < 160
    assert cuts[-1] == Gt


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        import paper_1705_09366_b200 as S
        from paper_1705_09366_b200.sharded import assemble, gather_slabs, rank_slab, validate_cuts
        w = synth.make_config("dengue")
        g = w.grid_kwargs()
        cuts = S.slab_cuts(w.G, 16, 5, 8.0, hist_T(w.points, g), world)
        validate_cuts(cuts, w.G[2], 16)
        # every rank derived the same cuts without communicating; verify that
        allc = [None] * world
        dist.all_gather_object(allc, cuts)
        assert all(c == cuts for c in allc)
        ref = oracle.stkde_pb(w.points, with_ambiguity=False, **g).vol
        t0, t1 = rank_slab(cuts, rank)
        slab = torch.from_numpy(np.ascontiguousarray(ref[:, :, t0:t1]))   # this rank's slab
        got = gather_slabs(slab, cuts, w.G, root=0)
        if rank == 0:
            full = assemble(got, cuts, w.G).numpy()
            assert np.array_equal(full, ref)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))


def _worker_x(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        import paper_1705_09366_b200 as S
        from paper_1705_09366_b200.sharded import assemble, gather_slabs, rank_slab, validate_cuts
        w = synth.make_config("dengue")
        g = w.grid_kwargs()
        hx = np.bincount(np.clip(np.floor(w.points[:, 0]).astype(np.int64), 0, w.G[0] - 1), minlength=w.G[0])
        cuts = S.xslab_cuts(w.G, 8.0, 5.0, hx, world)
        validate_cuts(cuts, w.G[0], 16)
        allc = [None] * world
        dist.all_gather_object(allc, cuts)
        assert all(c == cuts for c in allc)
        ref = oracle.stkde_pb(w.points, with_ambiguity=False, **g).vol
        x0, x1 = rank_slab(cuts, rank)
        slab = torch.from_numpy(np.ascontiguousarray(ref[x0:x1]))      # this rank's x-slab
        got = gather_slabs(slab, cuts, w.G, root=0, axis="x")
        if rank == 0:
            full = assemble(got, cuts, w.G, axis="x").numpy()
            assert np.array_equal(full, ref)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))


def test_gloo_world2_xslab_gather_assemble(S, oracle_mod):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker_x, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


def test_gloo_world2_gather_assemble(S, oracle_mod):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


def test_xslab_cuts_host():
    # stkde_xslab_cuts (host-only half of the x partition): multiples of 16, ordered, covering
    # [0, Gx), no empty part while nparts <= Gx/16, and more cuts where the points are
    import paper_1705_09366_b200 as S
    Gx, Gy, Gt = 1024, 512, 256
    uniform = [100] * Gx
    for n in (1, 2, 4, 8):
        c = S.xslab_cuts((Gx, Gy, Gt), 6.0, 4.0, uniform, n)
        assert c[0] == 0 and c[-1] == Gx and len(c) == n + 1
        assert all(b > a for a, b in zip(c[:-1], c[1:])) and all(x % 16 == 0 for x in c[:-1])
        widths = [b - a for a, b in zip(c[:-1], c[1:])]
        assert max(widths) - min(widths) <= 16          # uniform points: equal widths
    skew = [10 ** 6 if x < 128 else 1 for x in range(Gx)]  # compute-dominated mass in the first 128 columns
    c = S.xslab_cuts((Gx, Gy, Gt), 6.0, 4.0, skew, 4)
    assert c[1] <= 128 and c[2] <= 128


def _worker_handle(rank, world, port, q):
    # the direct gather's host protocol: the root's export is broadcast to every rank; row
    # offsets place each x-slab in the root's [Gx][Gy][Gt] float32 grid
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_1705_09366_b200.sharded import direct_row_offset, exchange_root_handle
        calls = []

        def export():
            calls.append(rank)
            return bytes(range(64)), 4096
        h, off = exchange_root_handle(rank, 1, export)
        assert h == bytes(range(64)) and off == 4096
        assert calls == ([1] if rank == 1 else [])          # only the root exports
        assert direct_row_offset(0, (64, 32, 16)) == 0
        assert direct_row_offset(5, (64, 32, 16)) == 5 * 32 * 16 * 4
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))


def test_gloo_world2_direct_gather_protocol():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker_handle, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
