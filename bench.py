#!/usr/bin/env python
"""STKDE (PB-SYM hot path) benchmark on B200 -- the driver contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config stress] [--impl reference]

One step = one full pass of the hot path (binning, work list, tile kernel) over
the workload's synthetic point set, producing the whole FP32 density grid
(N = 1) or this rank's time slab of it (N > 1, launched with torchrun, one
rank per GPU, cost-balanced Bt-aligned time slabs, no collective on the data
path).  Metric: point-voxel contributions per second (BASELINE.json), where
the contributions C are the exact gated (point, voxel) pairs, counted once by
the library's own count kernel outside the timed region.

Timing: W untimed warm-up steps; K timed steps, each bracketed by CUDA events
on the compute stream, with a 256 MiB L2 flush (untimed) between steps; barrier
+ synchronize on both sides; max over ranks.  `e2e` repeats the measurement
through the public API from pinned host memory: per step the points go H2D,
the grid (slab) comes back D2H, both inside the timed region.

--impl reference: the FP64 CPU oracle (oracle/) timed on this host's cores on
a bounded sample of the same workload (rank 0 only; other ranks exit 0).

--variant (default `fixed` is the driver's headline):
  adaptive  per-point bandwidths (stkde_compute_adaptive_slab) from
            stkde_synth.adaptive_bandwidths (Abramson square-root law on a pilot
            histogram, lambda in [0.25, 1]); C = the adaptive gated pairs.
  sweep     stkde_compute_sweep over (f hs, f ht), f in stkde_synth.SWEEP_FRACTIONS:
            one binning, one grid per bandwidth; C = sum over the grids.  N = 1 only.
            `separate_ms` times the same grids as separate plans + computes.
  f64       the FP64-output option (stkde_compute_slab_f64): every
            term in FP64 with Alg. 1's operation sequence, float64 grid; roofline against
            the FP64 pipe.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import stkde_synth as synth  # noqa: E402

METRIC = "point-voxel contributions/sec"
UNIT = "contributions/s"
FP32_NOMINAL_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12   # 74.4: SMs x FP32 lanes x 2 x max SM clock
FP64_NOMINAL_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12    # 37.2: SMs x FP64 lanes x 2 x max SM clock
ENGINES = {0: "SIMT FP32 FFMA2", 1: "mma.sync m16n8k16 3xFP16", 2: "tcgen05.mma kind::i8, exact S32",
           3: "short-window FP32 FFMA2 (window-offset dispatch)"}
KERNELS = {0: "stkde::k_tile<Bt=%d>", 1: "stkde::k_tile_mma<Bt=%d>", 2: "stkde::k_tile_tc<Bt=%d>",
           3: "stkde::k_tile_ws<Bt=%d>"}
# the arithmetic type of the contraction (not a precision claim; NUMERICS says what it means)
DTYPES = {0: "f32", 1: "f16", 2: "u8", 3: "f32"}
NUMERICS = {0: "FP32 FFMA2 accumulation, two-level summation",
            1: "3-term FP16 split (mma.sync m16n8k16), FP32 accumulation, two-level summation",
            2: "23-bit fixed-point factors as three u8 limbs (tcgen05.mma kind::i8), exact S32 accumulation, "
               "each voxel rounded from its exact int64 sum (int64 -> float, x scale); max |gpu - oracle| <= 9e-7 of max (DESIGN.md §5)",
            3: "FP32 FFMA2 accumulation of each point's temporal window, every voxel in candidate order (DESIGN.md §3.11)"}
NUMERICS_F64 = ("FP64 gates and factors with Alg. 1's operation sequence, fma accumulation in FP64, float64 grid; "
                "|gpu - oracle| <= 2 (n + 2) 2^-53 f per voxel, exact support (DESIGN.md §3.8)")
CONFIG_INDEX = {"tiny": 0, "dengue": 1, "social": 2, "ornith": 3, "stress": 4}
# oracle sample sizes for the cpu_baseline / reference legs (about 10-30 s of host work)
ORACLE_SAMPLE = {"tiny": 2000, "dengue": 11000, "social": 600000, "ornith": 1000000, "stress": 150000}
# per-step sample of the --impl reference arm (a few seconds per step, so K steps end in minutes)
REF_SAMPLE = {"tiny": 2000, "dengue": 11000, "social": 200000, "ornith": 200000, "stress": 20000}


def peaks():
    """(HBM GB/s, source), (dense bf16 TFLOP/s burst, source) from MEASURED_PEAKS.json, else the
    B200_PROFILING.md fallbacks."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    hbm, src = 6650.0, "fallback (B200_PROFILING.md)"
    bf16, bsrc = 1590.0, "fallback (B200_PROFILING.md)"
    if os.path.exists(p):
        try:
            d = json.load(open(p))
            hbm, src = float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
            bf16, bsrc = float(d["bf16_tflops"]), "measured (MEASURED_PEAKS.json, burst)"
        except Exception:
            pass
    return (hbm, src), (bf16, bsrc)


def host_cores():
    """Threads the oracle legs use (the cores this process may run on)."""
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def host_cpu():
    """{physical_cores, logical_cpus, model} of this host (lscpu's Core(s) per socket x
    Socket(s), else /proc/cpuinfo's distinct (physical id, core id) pairs)."""
    model, phys, logical = None, None, os.cpu_count()
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        kv = {a.strip(): b.strip() for a, b in (ln.split(":", 1) for ln in out.splitlines() if ":" in ln)}
        model = kv.get("Model name")
        if "Core(s) per socket" in kv and "Socket(s)" in kv:
            phys = int(kv["Core(s) per socket"]) * int(kv["Socket(s)"])
    except Exception:
        pass
    if phys is None or model is None:
        try:
            cores, m = set(), None
            pid = cid = None
            for ln in open("/proc/cpuinfo"):
                k, _, v = ln.partition(":")
                k, v = k.strip(), v.strip()
                if k == "model name":
                    m = m or v
                elif k == "physical id":
                    pid = v
                elif k == "core id":
                    cid = v
                elif not k and pid is not None:
                    cores.add((pid, cid))
                    pid = cid = None
            phys = phys or (len(cores) or None)
            model = model or m
        except Exception:
            pass
    return {"physical_cores": phys, "logical_cpus": logical, "model": model}


def cpu_baseline_dict(value, sample):
    d = {"value": value, "unit": UNIT, "cores": host_cores(), "kind": "oracle", "sample": sample}
    d.update({"host_" + k: v for k, v in host_cpu().items()})
    return d


# ----------------------------------------------------------------- clocks ---
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), "--query-gpu=" + self.FIELDS,
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # the first sample before the timed region starts (short regions then still have
            # one sample on each side: the samples bracket the region)
            t0 = time.time()
            while not self.lines and time.time() - t0 < 2.0:
                time.sleep(0.01)
            self.n0 = len(self.lines)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            n1, t0 = len(self.lines), time.time()
            while len(self.lines) <= n1 and time.time() - t0 < 2.0:   # one sample after the region
                time.sleep(0.01)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# -------------------------------------------------------------- reference ---
def run_oracle_sample(w, m, variant="fixed"):
    """The oracle as it stands on the first m points: (contributions, seconds)."""
    import oracle
    oracle.build()
    g = w.grid_kwargs()
    pts = np.ascontiguousarray(w.points[:m])
    t0 = time.perf_counter()
    if variant == "adaptive":
        bw = synth.adaptive_bandwidths(w)[:m]
        r = oracle.stkde_pb_adaptive(pts, bw, with_ambiguity=False, nthreads=host_cores(), **g)
        C = r.contributions
    elif variant == "sweep":
        C = 0
        for f in synth.SWEEP_FRACTIONS:
            r = oracle.stkde_pb(pts, with_ambiguity=False, nthreads=host_cores(),
                                **dict(g, hs=f * w.hs, ht=f * w.ht))
            C += r.contributions
    else:
        r = oracle.stkde_pb(pts, with_ambiguity=False, nthreads=host_cores(), **g)
        C = r.contributions
    dt = time.perf_counter() - t0
    return C, dt


def reference_main(args, w, rank):
    if rank != 0:
        return 0
    m = min(REF_SAMPLE[w.name], w.n)
    if args.variant == "sweep":
        m = max(m // len(synth.SWEEP_FRACTIONS), 1)
    sample = "first %d of %d points of the %s workload, full %dx%dx%d grid (FP64 oracle, PB form%s)" % (
        m, w.n, w.name, *w.G, "" if args.variant == "fixed" else ", " + args.variant)
    if args.warmup > 0:
        run_oracle_sample(w, min(m, 500), args.variant)
    vals, secs = [], []
    for _ in range(max(args.steps, 1)):
        C, dt = run_oracle_sample(w, m, args.variant)
        vals.append(C / dt)
        secs.append(dt)
    v = statistics.median(vals)
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(secs),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": config_dict(w, None, variant_config(args.variant)),
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "cpu_baseline": cpu_baseline_dict(v, sample)}
    print(json.dumps(out))
    return 0


def variant_config(variant):
    if variant == "adaptive":
        return {"variant": "adaptive bandwidth (DESIGN.md R15): stkde_synth.adaptive_bandwidths, lambda in [0.25, 1]"}
    if variant == "sweep":
        return {"variant": "multi-bandwidth sweep: (f hs, f ht), f in %s, one binning" % (list(synth.SWEEP_FRACTIONS),)}
    if variant == "f64":
        return {"variant": "FP64 output (stkde_compute_slab_f64): FP64 gates, factors and fma accumulation, "
                           "float64 grid (DESIGN.md §3.8)"}
    return {}


def config_dict(w, info, extra=None):
    d = {"workload": "%s (BASELINE.json configs[%d])" % (w.name, CONFIG_INDEX[w.name]), "n": w.n,
         "grid": list(w.G), "hs_voxels": w.hs / w.sres, "ht_voxels": w.ht / w.tres,
         "kernel": "printed (PAPER.md:132-133)"}
    if info:
        d["tile"] = [info["Bx"], info["By"], info["Bt"]]
    if extra:
        d.update(extra)
    return d


# --------------------------------------------------------------------- GPU ---
# collectives of the bench's own bookkeeping (counts, max-over-ranks times): NCCL on device
# tensors, or -- STKDE_BENCH_SHARED_GPU=1, the rehearsal of the N-rank path with every rank on
# one GPU, where NCCL refuses two ranks per device -- gloo on host copies
_GLOO = {"on": False}


def allreduce(t, op=None):
    import torch.distributed as dist
    op = dist.ReduceOp.SUM if op is None else op
    if _GLOO["on"]:
        c = t.cpu()
        dist.all_reduce(c, op=op)
        t.copy_(c)
    else:
        dist.all_reduce(t, op=op)


def direct_gather_ms(S, plan, pts, full, rank, local_rank, x0, x1, w, stream, barrier, dev):
    """The direct gather fused into the compute (stkde_ipc_*): each rank's tile kernel stores its
    x-slab straight into rank 0's grid over NVLink; one pass (binning + tiles) per step, the max
    over ranks (compare with ms_per_step, the same pass into the rank's own buffer)."""
    import torch
    import torch.distributed as dist
    from paper_1705_09366_b200.sharded import direct_row_offset, exchange_root_handle
    handle, root_off = exchange_root_handle(rank, 0, lambda: S.ipc_handle(full))
    peer, why = None, ""
    try:
        peer = S.IpcMapping(handle, local_rank) if rank != 0 else None
    except Exception as e:  # pragma: no cover - hardware-specific
        why = repr(e)[:200]
    ok = torch.tensor([0 if why else 1], dtype=torch.int32, device=dev)
    allreduce(ok, op=dist.ReduceOp.MIN)         # every rank mapped the root's grid, or none times
    if not int(ok.item()):
        if peer is not None:
            peer.close()
        return {"error": why or "another rank could not map rank 0's grid"}
    try:
        ptr = (full.data_ptr() if rank == 0 else peer.ptr(root_off)) + direct_row_offset(x0, w.G)

        def direct():
            if x1 > x0:
                plan.compute_xslab_to(pts, x0, x1, ptr, n_norm=w.n, stream=stream)
        direct()
        barrier()
        dd = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(3)]
        for a_, b_ in dd:
            a_.record(stream)
            direct()
            b_.record(stream)
        barrier()
        d_ms = torch.tensor([sum(a_.elapsed_time(b_) for a_, b_ in dd) / len(dd)], dtype=torch.float64, device=dev)
        allreduce(d_ms, op=dist.ReduceOp.MAX)
    finally:
        if peer is not None:
            peer.close()
    return {"ms_per_step_into_root": float(d_ms.item()),
            "how": "stkde_compute_xslab into rank 0's grid mapped with stkde_ipc_open: the epilogue's stores "
                   "cross NVLink while the rank computes (no separate gather)"}


def gpu_main(args, w, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_1705_09366_b200 as S

    # STKDE_BENCH_SHARED_GPU=1: a rehearsal of the N-rank control flow on a box with fewer GPUs
    # than ranks (ranks share devices round-robin, gloo for the bookkeeping collectives, the
    # library's NCCL gather skipped); its times are not a scaling measurement and the line says so
    shared = world > 1 and os.environ.get("STKDE_BENCH_SHARED_GPU") == "1"
    gpu_idx = local_rank
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if shared:
        local_rank = local_rank % torch.cuda.device_count()
    if vis:
        gpu_idx = vis.split(",")[local_rank]
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    if world > 1:
        _GLOO["on"] = shared
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    g = w.grid_kwargs()
    variant = args.variant
    if variant == "sweep" and world > 1:
        if rank == 0:
            print(json.dumps({"variant": "sweep", "unavailable": "the sweep bench runs on one GPU"}))
        dist.destroy_process_group()
        return 0
    stream = torch.cuda.Stream(dev)
    plan = S.Plan(max_n=w.n, device=local_rank, **g)
    info = plan.info()
    pts = torch.from_numpy(w.points).to(dev)
    bw_host = synth.adaptive_bandwidths(w) if variant == "adaptive" else None
    bw = torch.from_numpy(bw_host).to(dev) if bw_host is not None else None
    fr = synth.SWEEP_FRACTIONS
    sw_hs, sw_ht = [f * w.hs for f in fr], [f * w.ht for f in fr]
    # N > 1: the fixed and adaptive variants split the grid into cost-balanced X-slabs
    # (stkde_compute_[adaptive_]xslab: the slab's tiles are the full grid's, so the work splits
    # without overhead)
    xsplit = world > 1 and variant in ("fixed", "adaptive")
    x0, x1 = 0, w.G[0]
    with torch.cuda.stream(stream):
        if xsplit:
            xcuts = plan.xslab_partition(pts, world, stream=stream)
            x0, x1 = xcuts[rank], xcuts[rank + 1]
            cuts = [0, w.G[2]]
        else:
            cuts = plan.slab_partition(pts, world, stream=stream) if world > 1 else [0, w.G[2]]
        t0, t1 = cuts[0 if xsplit else rank], cuts[1 if xsplit else rank + 1]
        if xsplit and variant == "adaptive":   # the metric's C is the whole grid's: count it on rank 0
            C = int(plan.count_contributions_adaptive(pts, bw, 0, w.G[2], stream=stream).item()) if rank == 0 else 0
        elif xsplit:                           # this rank's own contributions (its x-slab), exactly
            C = int(plan.count_contributions_box(pts, x0, x1, 0, w.G[2], stream=stream).item()) if x1 > x0 else 0
        elif t1 <= t0:
            C = 0
        elif variant == "adaptive":
            C = int(plan.count_contributions_adaptive(pts, bw, t0, t1, stream=stream).item())
        elif variant == "sweep":
            C = 0
            for hs_k, ht_k in zip(sw_hs, sw_ht):
                with S.Plan(max_n=w.n, device=local_rank, **dict(g, hs=hs_k, ht=ht_k)) as q:
                    C += int(q.count_contributions(pts, t0, t1, stream=stream).item())
        else:
            C = int(plan.count_contributions(pts, t0, t1, stream=stream).item())
    Ct = torch.tensor([C], dtype=torch.int64, device=dev)
    if world > 1:
        allreduce(Ct)
    C_total = int(Ct.item())
    C_own = C if not (xsplit and variant == "adaptive") else None   # exact per-rank count (None: estimate)
    odt = torch.float64 if variant == "f64" else torch.float32
    out = (torch.empty((max(x1 - x0, 1), w.G[1], w.G[2]), dtype=odt, device=dev) if xsplit else
           torch.empty((w.G[0], w.G[1], max(t1 - t0, 1)), dtype=odt, device=dev))
    outs = [out] + [torch.empty_like(out) for _ in fr[1:]] if variant == "sweep" else [out]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def run(p_pts, p_bw):
        if t1 <= t0:
            return
        if variant == "adaptive" and xsplit:
            if x1 > x0:
                plan.compute_adaptive_xslab(p_pts, p_bw, x0, x1, n_norm=w.n, out=out, stream=stream)
        elif variant == "adaptive":
            plan.compute_adaptive_slab(p_pts, p_bw, t0, t1, n_norm=w.n, out=out, stream=stream)
        elif variant == "sweep":
            plan.compute_sweep(p_pts, sw_hs, sw_ht, outs=outs, stream=stream)
        elif variant == "f64":
            plan.compute_f64(p_pts, t0, t1, n_norm=w.n, out=out, stream=stream)
        elif xsplit:
            if x1 > x0:
                plan.compute_xslab(p_pts, x0, x1, n_norm=w.n, out=out, stream=stream)
        else:
            plan.compute_slab(p_pts, t0, t1, n_norm=w.n, out=out, stream=stream)

    # fixed variant: the step is ONE CUDA-graph launch of the captured pass (the rank's slab)
    # (stkde_graph_create: binning, work list and tile kernel, ~20 kernels) -- the small grids
    # are launch-bound otherwise.  Same kernels, same work; --no-graph launches them one by one.
    graph = None
    if variant == "fixed" and not args.no_graph and t1 > t0:
        with torch.cuda.stream(stream):
            if xsplit:
                graph = plan.graph_xslab(pts, x0, x1, n_norm=w.n, out=out) if x1 > x0 else None
            else:
                graph = plan.graph(pts, out=out, t_begin=t0, t_end=t1, n_norm=w.n)

    def step():
        if graph is not None:
            graph.launch(stream)
        else:
            run(pts, bw)

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
    barrier()
    own = plan.info()["last_own_launches"]
    cub = plan.info()["last_cub_calls"]
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    plan.mma_stats()                            # reset the issued-MMA counters (tcgen05 engine)
    plan.enable_kernel_timing(True)
    with ClockSampler(gpu_idx) as clk:
        barrier()
        with torch.cuda.stream(stream):
            for e0, e1 in ev:
                flush.fill_(1)                  # untimed 256 MiB L2 flush
                e0.record(stream)
                step()
                e1.record(stream)
        barrier()
    ms_steps = [a.elapsed_time(b) for a, b in ev]
    if graph is not None:
        # the tile kernel's launch duration: the same steps launched one by one (a graph
        # replays no per-launch event records), CUDA events on the compute stream
        kms, klaunch = plan.kernel_ms()          # (resets nothing recorded inside the graph)
        plan.enable_kernel_timing(True)
        plan.mma_stats()                        # issued-MMA counters: these K launches only
        with torch.cuda.stream(stream):
            for _ in range(args.steps):
                flush.fill_(1)
                run(pts, bw)
        barrier()
    kms, klaunch = plan.kernel_ms()
    plan.enable_kernel_timing(False)
    mma_cols, mma_kblocks = plan.mma_stats()
    # per-phase device time (stkde_plan_enable_phase_timing: CUDA events at every phase end on
    # the compute stream), from a separate untimed pass of the same steps launched one by one
    plan.enable_phase_timing(True)
    with torch.cuda.stream(stream):
        for _ in range(args.steps):
            flush.fill_(1)
            run(pts, bw)
    barrier()
    ph_ms, ph_calls = plan.phase_ms()
    plan.enable_phase_timing(False)
    phases = {k: round(v / max(args.steps, 1), 4) for k, v in ph_ms.items() if v > 0}
    ms = sum(ms_steps) / len(ms_steps)
    kernel_ms = kms / max(args.steps, 1)          # tile-kernel time per step (all its launches)
    vals = torch.tensor([ms, kernel_ms], dtype=torch.float64, device=dev)
    if world > 1:
        allreduce(vals, op=dist.ReduceOp.MAX)
    ms_max, kernel_ms_max = float(vals[0]), float(vals[1])

    # ---- e2e through the public API: pinned host points in, grid (slab) out ----
    host_pts = torch.from_numpy(w.points).pin_memory()
    host_bw = torch.from_numpy(bw_host).pin_memory() if bw_host is not None else None
    host_outs = None
    e2e_steps = max(1, min(args.steps, 10))
    # fixed variant: the grid is produced as Bt-layer T-slabs (stkde_compute_slab) and slab k's
    # device->host copy runs on a second stream while slab k+1 is computed
    pipe = None
    xpipe = None
    if xsplit and x1 > x0:
        # this rank's rows in 4 x sub-slabs (multiples of 16): sub-slab k's D2H into its rows of
        # one pinned buffer overlaps sub-slab k+1's compute
        step16 = max(16, ((x1 - x0) // 4 + 15) // 16 * 16)
        xs = list(range(x0, x1, step16)) + [x1]
        host_full = torch.empty(tuple(out.shape), dtype=torch.float32).pin_memory()
        xpipe = [(a, b) for a, b in zip(xs[:-1], xs[1:])]
        host_outs = [host_full]
        copy_stream = torch.cuda.Stream(dev)
        slab_ev = [torch.cuda.Event() for _ in xpipe]
    elif variant == "fixed" and t1 > t0:
        Bt = info["Bt"]
        sc = list(range(t0, t1, Bt)) + [t1]
        pipe = [(a, b, torch.empty((w.G[0], w.G[1], b - a), dtype=torch.float32, device=dev),
                 torch.empty((w.G[0], w.G[1], b - a), dtype=torch.float32).pin_memory())
                for a, b in zip(sc[:-1], sc[1:])]
        host_outs = [hb for _, _, _, hb in pipe]
        copy_stream = torch.cuda.Stream(dev)
        slab_ev = [torch.cuda.Event() for _ in pipe]
    if host_outs is None:
        host_outs = [torch.empty(tuple(out.shape), dtype=out.dtype).pin_memory() for _ in outs]
    barrier()
    eb, ee = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        eb.record(stream)
        for _ in range(e2e_steps):
            dpts = host_pts.to(dev, non_blocking=True)
            dbw = host_bw.to(dev, non_blocking=True) if host_bw is not None else None
            if xpipe is not None:
                stream.wait_stream(copy_stream)
                for (a, b), ev in zip(xpipe, slab_ev):
                    if variant == "adaptive":
                        plan.compute_adaptive_xslab(dpts, dbw, a, b, n_norm=w.n, out=out[a - x0:b - x0], stream=stream)
                    else:
                        plan.compute_xslab(dpts, a, b, n_norm=w.n, out=out[a - x0:b - x0], stream=stream)
                    ev.record(stream)
                    copy_stream.wait_event(ev)
                    with torch.cuda.stream(copy_stream):
                        host_full[a - x0:b - x0].copy_(out[a - x0:b - x0], non_blocking=True)
                stream.wait_stream(copy_stream)
            elif pipe is None:
                run(dpts, dbw)
                for ho, o in zip(host_outs, outs):
                    ho.copy_(o, non_blocking=True)
            else:
                stream.wait_stream(copy_stream)        # last step's copies left the slab buffers
                for (a, b, db, hb), ev in zip(pipe, slab_ev):
                    plan.compute_slab(dpts, a, b, n_norm=w.n, out=db, stream=stream)
                    ev.record(stream)
                    copy_stream.wait_event(ev)
                    with torch.cuda.stream(copy_stream):
                        hb.copy_(db, non_blocking=True)
                stream.wait_stream(copy_stream)
        ee.record(stream)
    barrier()
    e2e_ms = torch.tensor([eb.elapsed_time(ee) / e2e_steps], dtype=torch.float64, device=dev)
    if world > 1:
        allreduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_ms = float(e2e_ms.item())
    h2d = (w.points.nbytes + (bw_host.nbytes if bw_host is not None else 0)) * world
    esz = out.element_size()
    d2h = w.G[0] * w.G[1] * w.G[2] * esz * len(outs)

    # sweep: the same grids as separate plans + computes (what the one binning saves)
    separate_ms = None
    if variant == "sweep":
        qs = [S.Plan(max_n=w.n, device=local_rank, **dict(g, hs=a, ht=b)) for a, b in zip(sw_hs, sw_ht)]
        def sep():
            for q, o in zip(qs, outs):
                q.compute(pts, out=o, stream=stream)
        with torch.cuda.stream(stream):
            for _ in range(args.warmup):
                sep()
        barrier()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(max(1, min(args.steps, 10)))]
        with torch.cuda.stream(stream):
            for a, b in evs:
                flush.fill_(1)
                a.record(stream)
                sep()
                b.record(stream)
        barrier()
        separate_ms = sum(a.elapsed_time(b) for a, b in evs) / len(evs)
        for q in qs:
            q.close()

    # ---- roofline of the dominant kernel (the tile kernel) ----
    (hbm_peak, hbm_src), (bf16_peak, bf16_src) = peaks()
    grid_bytes = (x1 - x0) * w.G[1] * (t1 - t0) * esz * len(outs)
    t_hbm = grid_bytes / (hbm_peak * 1e9)
    # this rank's own work (exact for the fixed variant; the adaptive x-slab count is the global
    # one, so its per-rank share is estimated as C / N over the cost-balanced cuts)
    C_rank = C_own if C_own is not None else C_total / world
    t_fp32 = 2.0 * C_rank / (FP32_NOMINAL_TFLOPS * 1e12)
    if variant == "f64" and 2.0 * C_rank / (FP64_NOMINAL_TFLOPS * 1e12) >= t_hbm:
        ach = 2.0 * C_rank / (kernel_ms * 1e-3) / 1e12
        roof = {"bound": "alu", "achieved": ach, "peak": FP64_NOMINAL_TFLOPS, "unit": "TFLOP/s (FP64)",
                "frac": ach / FP64_NOMINAL_TFLOPS,
                "peak_source": "derived: 148 SMs x 64 FP64 lanes x 2 FLOP x 1.965 GHz (DESIGN.md §3.8); "
                               "tools/fma_peak measured 36.5 TFLOP/s DFMA"}
    elif t_fp32 >= t_hbm and variant != "f64":
        ach = 2.0 * C_rank / (kernel_ms * 1e-3) / 1e12
        roof = {"bound": "alu", "achieved": ach, "peak": FP32_NOMINAL_TFLOPS, "unit": "TFLOP/s",
                "frac": ach / FP32_NOMINAL_TFLOPS,
                "peak_source": "derived: 148 SMs x 128 FP32 lanes x 2 FLOP x 1.965 GHz (DESIGN.md §4); "
                               "tools/fma_peak measured 74.2 TFLOP/s FFMA2"}
    else:
        ach = grid_bytes / (kernel_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak,
                "peak_source": hbm_src}
    roof["traffic"] = profile_traffic(w.name, info["engine"], variant)
    roof["kernel"] = "stkde::k_tile_f64" if variant == "f64" else KERNELS[info["engine"]] % info["Bt"]
    roof["kernel_ms"] = kernel_ms_max
    roof["algorithmic"] = {"flops": 2 * C_rank, "bytes": grid_bytes,
                           "per_unit": "2 FLOP per contribution (one FMA acc += K_s*K_t), %d B per voxel written once"
                                       % esz}
    # the tensor pipe's own roofline (tcgen05 engine): int8 ops the kernel issued per launch
    # (7 MMAs of 128 x N x 32 per k-block, 2 ops per MAC) against the dense int8 peak
    # = 2 x the measured dense bf16 peak (the guide's nominal int8:bf16 ratio on sm_100)
    roof_tc = None
    if info["engine"] == 2 and mma_kblocks > 0:
        ops = 7 * 2 * 128 * 32 * mma_cols / args.steps
        ach_t = ops / (kernel_ms * 1e-3) / 1e12
        roof_tc = {"bound": "tensor", "achieved": ach_t, "peak": 2 * bf16_peak, "unit": "TOPS (int8)",
                   "frac": ach_t / (2 * bf16_peak), "peak_source": "2 x " + bf16_src,
                   "kblocks_per_launch": mma_kblocks / args.steps,
                   "mean_mma_n": mma_cols / mma_kblocks,
                   # contributions / (128 x N x 32 products per k-block): the share of the
                   # tile contraction that is inside some disc and window
                   "useful_fraction": C_rank / (128 * 32 * mma_cols / args.steps)}

    if world > 1:       # the line carries rank 0's roofline; the slowest rank's fraction too
        fr_t = torch.tensor([roof["frac"]], dtype=torch.float64, device=dev)
        allreduce(fr_t, op=dist.ReduceOp.MIN)
        roof["rank"] = 0
        roof["frac_min_over_ranks"] = float(fr_t.item())

    # ---- optional whole-grid gather (outside the timed region, reported separately) ----
    # x-slabs are contiguous row blocks of the [Gx][Gy][Gt] layout: rank r's slab lands in rows
    # [cut_r, cut_r+1) of rank 0's grid by one NCCL recv per rank (point-to-point over NVLink)
    gather = None
    if world > 1 and xsplit and variant == "fixed":
        full = torch.empty(tuple(w.G), dtype=torch.float32, device=dev) if rank == 0 else None
        if shared:   # NCCL refuses two ranks on one device: the rehearsal skips the library gather
            gather = {"skipped": "STKDE_BENCH_SHARED_GPU rehearsal (ranks share a GPU; NCCL needs one device per rank)"}
        else:
            # the library's own NCCL communicator (stkde_plan_comm_init), id shipped over the group
            uid = [S.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            plan.comm_init(world, rank, uid[0])
            slab = out[:max(x1 - x0, 0)]

            def do_gather():
                with torch.cuda.stream(stream):
                    plan.gather_xslab(slab, xcuts, 0, full, stream=stream)
            do_gather()                                   # warm-up (NCCL P2P connection setup)
            barrier()
            gb_, ge_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            gb_.record(stream)
            do_gather()
            ge_.record(stream)
            barrier()
            g_ms = torch.tensor([gb_.elapsed_time(ge_)], dtype=torch.float64, device=dev)
            allreduce(g_ms, op=dist.ReduceOp.MAX)
            gbytes = (w.G[0] - (x1 - x0 if rank == 0 else 0)) * w.G[1] * w.G[2] * 4
            gather = {"ms": float(g_ms.item()), "bytes_to_root": gbytes,
                      "how": "stkde_gather_xslab: NCCL send/recv group inside the library, each rank's x-slab "
                             "received in place into its rows of rank 0's grid",
                      "timed_in_value": False}
        # the direct gather fused into the compute (stkde_ipc_*): each rank's tile kernel stores its
        # x-slab straight into rank 0's grid over NVLink; one pass (binning + tiles) per step, the
        # max over ranks, against the same pass into the rank's own buffer (ms_per_step)
        # (a failure here is recorded in the line, never loses it; the path itself is tested
        # bitwise on one GPU by tests/test_gpu_direct_gather.py)
        try:
            gather["direct"] = direct_gather_ms(S, plan, pts, full, rank, local_rank, x0, x1, w, stream, barrier, dev)
        except Exception as e:  # pragma: no cover - hardware-specific
            gather["direct"] = {"error": repr(e)[:200]}
        del full

    result = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            m = min(ORACLE_SAMPLE[w.name], w.n)
            if variant == "sweep":
                m = max(m // len(fr), 1)
            Cs, dt = run_oracle_sample(w, m, variant)
            cpu = cpu_baseline_dict(Cs / dt, "first %d of %d points, full %dx%dx%d grid, FP64 oracle (PB form%s), %.1f s"
                                    % (m, w.n, *w.G, "" if variant == "fixed" else ", " + variant, dt))
        result = {
            "metric": METRIC, "value": C_total / (ms_max * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": "f64" if variant == "f64" else DTYPES[info["engine"]],
            "numerics": NUMERICS_F64 if variant == "f64" else NUMERICS[info["engine"]], "data": "synthetic",
            "config": config_dict(w, info, dict(variant_config(variant), **{
                "contributions": C_total, "ms_per_grid": ms_max / len(outs),
                "parallelism": ("x-slab x%d" if xsplit else "time-slab x%d") % world,
                "slab_cuts": xcuts if xsplit else cuts,
                "l2": "flushed between timed steps (256 MiB write, untimed)",
                "launch": "one CUDA graph per step (stkde_graph_launch)" if graph is not None else "kernel by kernel",
                "inputs_resident": True})),
            "e2e": {"value": C_total / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                    "pipeline": ("%d x sub-slabs per rank; D2H of sub-slab k overlaps the compute of k+1"
                                 % len(xpipe)) if xpipe else
                                ("%d T-slabs of Bt layers; D2H of slab k overlaps the compute of slab k+1"
                                 % len(pipe)) if pipe else "compute, then D2H"},
            "gpu_launches": own * args.steps,
            "library_launches": {"cub_calls": cub * args.steps},
            "clocks": clk.summary(),
            "roofline": roof,
            "roofline_tensor": roof_tc,
            "phases_ms_per_step": phases,
            "engine": "FP64 gather tiles (stkde_tile_f64.cu)" if variant == "f64" else ENGINES[info["engine"]],
            "cpu_baseline": cpu,
        }
        if variant != "fixed":
            result["variant"] = variant
        if separate_ms is not None:
            result["separate_ms"] = separate_ms
        if gather is not None:
            result["gather"] = gather
        if shared:
            result["rehearsal"] = ("STKDE_BENCH_SHARED_GPU=1: %d ranks shared %d GPU(s); the N-rank control flow "
                                   "on hardware, NOT a scaling measurement" % (world, torch.cuda.device_count()))
        print(json.dumps(result))
    plan.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def profile_traffic(name, engine, variant="fixed"):
    """dram__bytes_read.sum + dram__bytes_write.sum per step of the tile kernel from the
    committed ncu --set full capture of this workload and engine (profiles/traffic.json)."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        try:
            key = "%s/engine%d" % (name, engine) + ("" if variant == "fixed" else "/" + variant)
            return json.load(open(p)).get(key)
        except Exception:
            return None
    return None


def free_port():
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def self_launch(args):
    """--gpus N > 1 without a torchrun environment: start N ranks (one per GPU) under
    torch.distributed.run on this node and pass rank 0's JSON line through."""
    if not args.dry_run:
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus and os.environ.get("STKDE_BENCH_SHARED_GPU") != "1":
            print(json.dumps({"n_gpus": args.gpus, "error": "--gpus %d but only %d CUDA device(s) visible"
                              % (args.gpus, have)}))
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=dict(os.environ, STKDE_BENCH_LAUNCHED="1"))


def dry_main(args, w, rank, world):
    """--dry-run: the N-rank control flow of the bench on CPU (gloo, no CUDA): process group,
    cost-balanced x-slab cuts from the library's host-only partition (stkde_xslab_cuts),
    per-rank work, barrier + max-over-ranks timing, one JSON line from rank 0.  The per-rank
    'work' is a stand-in (its slab's point count), not the method: tests/test_bench_cpu.py."""
    import torch
    import torch.distributed as dist

    import paper_1705_09366_b200 as S
    if world > 1:
        dist.init_process_group("gloo")
    g = w.grid_kwargs()
    X = np.clip(np.floor((w.points[:, 0].astype(np.float64) - g["x0"]) / g["sres"]).astype(np.int64), 0, w.G[0] - 1)
    hist = np.bincount(X, minlength=w.G[0]).astype(np.int64)
    cuts = S.xslab_cuts(w.G, w.hs / w.sres, w.ht / w.tres, hist, world)
    x0, x1 = cuts[rank], cuts[rank + 1]
    mine = torch.tensor([int(((X >= x0) & (X < x1)).sum())], dtype=torch.int64)
    if world > 1:
        dist.all_reduce(mine)
    ms = []
    for _ in range(args.warmup + args.steps):
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        _ = int(((X >= x0) & (X < x1)).sum())
        if world > 1:
            dist.barrier()
        ms.append(1e3 * (time.perf_counter() - t0))
    v = torch.tensor([statistics.mean(ms[args.warmup:])], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"dry_run": True, "metric": METRIC, "n_gpus": world, "steps": args.steps,
                          "warmup": args.warmup, "ms_per_step": float(v.item()), "backend": "gloo",
                          "config": {"workload": w.name, "parallelism": "x-slab x%d" % world, "slab_cuts": cuts,
                                     "points_total": int(mine.item())}}))
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="stress", choices=sorted(CONFIG_INDEX))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--variant", default="fixed", choices=["fixed", "adaptive", "sweep", "f64"])
    ap.add_argument("--no-graph", action="store_true",
                    help="launch the pass kernel by kernel instead of one CUDA-graph launch per step")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU-only: the N-rank control flow over gloo, no CUDA (tests)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and not os.environ.get("STKDE_BENCH_LAUNCHED"):
        return self_launch(args)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if rank == 0:
            print(json.dumps({"n_gpus": args.gpus, "error": "--gpus %d but WORLD_SIZE %d" % (args.gpus, world)}))
        return 2
    w = synth.make_config(args.config)
    if args.dry_run:
        return dry_main(args, w, rank, world)
    if args.impl == "reference":
        return reference_main(args, w, rank)
    return gpu_main(args, w, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
