"""Per-phase timing / NVTX and the library's NCCL gather, on one GPU through the C ABI.

Phase timing: every enqueued phase is charged, the phases of a call sum
to its device time, the tcgen05 engine has no radix-sort phase (counting sort) while
the FP64 path does, and graph capture records nothing.  NCCL gather:
a one-rank communicator exercises the library's group of send/recv (x-slabs: the root's
own slab travels through NCCL to itself unless it is already in place) and the strided
time-slab unpack; the results must be bitwise equal to the computed grid.  More ranks
than GPUs are not emulated on one device (B200_PROFILING.md): the multi-rank control
flow of the slab drivers is covered on the CPU (tests/test_sharded_cpu.py).
"""
import numpy as np
import pytest

import stkde_synth as synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1705_09366_b200 as S
    S.load_library()
    return S


def _dengue(S):
    w = synth.make_config("dengue")
    pts = torch.from_numpy(w.points).cuda()
    return w, pts


def test_phase_timing_tc(S):
    w, pts = _dengue(S)
    with S.Plan(max_n=w.n, device=0, **w.grid_kwargs()) as p:
        out = p.compute(pts)                       # warm-up
        torch.cuda.synchronize()
        p.enable_phase_timing(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        K = 5
        e0.record()
        for _ in range(K):
            p.compute(pts, out=out)
        e1.record()
        ms, calls = p.phase_ms()
        total = e0.elapsed_time(e1)
        assert calls == K
        for ph in ("prep", "scan", "scatter", "chords", "worklist", "tiles"):
            assert ms[ph] > 0, (ph, ms)
        assert ms["sort"] == 0 and ms["gather"] == 0, ms        # counting sort; no gather
        s = sum(ms.values())
        # the phases tile each call: their sum is the calls' device time minus the gaps
        # between calls (host enqueue), never more than the bracketing interval
        assert s <= total * 1.02 + 0.01, (s, total)
        assert s >= 0.5 * total, (s, total)
        assert ms["tiles"] == max(ms.values())
        # off: nothing more is charged
        p.enable_phase_timing(False)
        p.compute(pts, out=out)
        ms2, calls2 = p.phase_ms()
        assert calls2 == 0 and sum(ms2.values()) == 0


def test_phase_timing_f64_has_sort(S):
    w, pts = _dengue(S)
    with S.Plan(max_n=w.n, device=0, **w.grid_kwargs()) as p:
        p.enable_phase_timing(True)
        p.compute_f64(pts)
        ms, calls = p.phase_ms()
        assert calls == 1
        assert ms["sort"] > 0 and ms["tiles"] > 0 and ms["chords"] == 0, ms


def test_phase_timing_skips_graph_capture(S):
    w, pts = _dengue(S)
    with S.Plan(max_n=w.n, device=0, **w.grid_kwargs()) as p:
        ref = p.compute(pts).clone()
        p.enable_phase_timing(True)
        g = p.graph(pts)
        for _ in range(3):
            g.launch()
        torch.cuda.synchronize()
        ms, calls = p.phase_ms()
        assert calls == 0 and sum(ms.values()) == 0
        assert torch.equal(g.out, ref)
        g.close()


def test_phase_timing_ring_wraps(S):
    # more marks than the 4096-event ring: the ring folds and keeps counting
    g = dict(x0=0.0, y0=0.0, t0=0.0, sres=1.0, tres=1.0, Gx=16, Gy=8, Gt=16, hs=2.0, ht=2.0)
    pts = torch.tensor([[8.0, 4.0, 8.0]], device="cuda")
    with S.Plan(max_n=1, device=0, **g) as p:
        out = p.compute(pts)
        p.enable_phase_timing(True)
        K = 700                                    # 7 marks per call -> 4900 marks
        for _ in range(K):
            p.compute(pts, out=out)
        ms, calls = p.phase_ms()
        assert calls == K
        assert all(ms[ph] > 0 for ph in ("prep", "scan", "scatter", "chords", "worklist", "tiles"))


def _comm1(S, p):
    uid = S.nccl_unique_id()
    assert len(uid) == 128
    p.comm_init(1, 0, uid)


def test_nccl_gather_xslab_one_rank(S):
    w, pts = _dengue(S)
    with S.Plan(max_n=w.n, device=0, **w.grid_kwargs()) as p:
        ref = p.compute(pts)
        _comm1(S, p)
        Gx = w.G[0]
        slab = p.compute_xslab(pts, 0, Gx)
        full = torch.full(w.G, -1.0, device="cuda")
        p.enable_phase_timing(True)
        p.gather_xslab(slab, [0, Gx], 0, full)      # through NCCL (root to itself)
        ms, calls = p.phase_ms()
        assert torch.equal(full, ref)
        assert calls == 1 and ms["gather"] > 0
        # already in place: nothing to move
        p.gather_xslab(full, [0, Gx], 0, full)
        assert torch.equal(full, ref)


def test_nccl_gather_slab_one_rank(S):
    w, pts = _dengue(S)
    with S.Plan(max_n=w.n, device=0, **w.grid_kwargs()) as p:
        ref = p.compute(pts)
        _comm1(S, p)
        Gt = w.G[2]
        slab = p.compute_slab(pts, 0, Gt)
        full = torch.full(w.G, -1.0, device="cuda")
        p.gather_slab(slab, [0, Gt], 0, full)       # root's own slab: the unpack kernel
        torch.cuda.synchronize()
        assert torch.equal(full, ref)


def test_nccl_gather_errors(S):
    w, pts = _dengue(S)
    with S.Plan(max_n=w.n, device=0, **w.grid_kwargs()) as p:
        slab = p.compute(pts)
        full = torch.empty(w.G, device="cuda")
        with pytest.raises(S.StkdeError) as e:     # no communicator yet
            p.gather_xslab(slab, [0, w.G[0]], 0, full)
        assert e.value.code == S.STKDE_EINVAL
        _comm1(S, p)
        for cuts, root in (([0, w.G[0] - 1], 0), ([1, w.G[0]], 0), ([0, w.G[0]], 1)):
            with pytest.raises(S.StkdeError) as e:
                p.gather_xslab(slab, cuts, root, full)
            assert e.value.code == S.STKDE_EINVAL
        with pytest.raises(S.StkdeError):           # no destination on the root
            p.gather_slab(slab, [0, w.G[2]], 0, None)
        with pytest.raises(S.StkdeError):
            p.comm_init(2, 2, S.nccl_unique_id())   # rank outside [0, nranks)


def test_sharded_driver_gather_world1(S):
    # the per-rank driver's library gather at world size 1 (axis x and t)
    import os
    import torch.distributed as dist
    from paper_1705_09366_b200.sharded import ShardedSTKDE
    w, pts = _dengue(S)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29613")
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        with S.Plan(max_n=w.n, device=0, **w.grid_kwargs()) as p:
            ref = p.compute(pts)
        for axis in ("x", "t"):
            d = ShardedSTKDE(pts, grid=w.grid_kwargs(), rank=0, world=1, axis=axis)
            d.init_comm()
            full = d.gather(d.compute())
            torch.cuda.synchronize()
            assert torch.equal(full, ref), axis
            d.close()
    finally:
        dist.destroy_process_group()
