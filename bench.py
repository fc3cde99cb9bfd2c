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
ENGINES = {0: "SIMT FP32 FFMA2", 1: "mma.sync m16n8k16 3xFP16", 2: "tcgen05.mma kind::i8, exact S32"}
KERNELS = {0: "stkde::k_tile<Bt=%d>", 1: "stkde::k_tile_mma<Bt=%d>", 2: "stkde::k_tile_tc<Bt=%d>"}
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
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


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
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
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
def run_oracle_sample(w, m):
    import oracle
    oracle.build()
    g = w.grid_kwargs()
    pts = np.ascontiguousarray(w.points[:m])
    t0 = time.perf_counter()
    r = oracle.stkde_pb(pts, with_ambiguity=False, nthreads=host_cores(), **g)
    dt = time.perf_counter() - t0
    return r.contributions, dt


def reference_main(args, w, rank):
    if rank != 0:
        return 0
    m = min(REF_SAMPLE[w.name], w.n)
    sample = "first %d of %d points of the %s workload, full %dx%dx%d grid (FP64 oracle, PB form)" % (
        m, w.n, w.name, *w.G)
    if args.warmup > 0:
        run_oracle_sample(w, min(m, 500))
    vals, secs = [], []
    for _ in range(max(args.steps, 1)):
        C, dt = run_oracle_sample(w, m)
        vals.append(C / dt)
        secs.append(dt)
    v = statistics.median(vals)
    cores = host_cores()
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(secs),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": config_dict(w, None),
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample}}
    print(json.dumps(out))
    return 0


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
def gpu_main(args, w, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_1705_09366_b200 as S

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    g = w.grid_kwargs()
    stream = torch.cuda.Stream(dev)
    plan = S.Plan(max_n=w.n, device=local_rank, **g)
    info = plan.info()
    pts = torch.from_numpy(w.points).to(dev)
    with torch.cuda.stream(stream):
        cuts = plan.slab_partition(pts, world, stream=stream) if world > 1 else [0, w.G[2]]
        t0, t1 = cuts[rank], cuts[rank + 1]
        C = int(plan.count_contributions(pts, t0, t1, stream=stream).item()) if t1 > t0 else 0
    Ct = torch.tensor([C], dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(Ct)
    C_total = int(Ct.item())
    out = torch.empty((w.G[0], w.G[1], max(t1 - t0, 1)), dtype=torch.float32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step():
        if t1 > t0:
            plan.compute_slab(pts, t0, t1, n_norm=w.n, out=out, stream=stream)

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
    gpu_idx = local_rank
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        gpu_idx = vis.split(",")[local_rank]
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
    kms, klaunch = plan.kernel_ms()
    plan.enable_kernel_timing(False)
    mma_cols, mma_kblocks = plan.mma_stats()
    ms = sum(ms_steps) / len(ms_steps)
    kernel_ms = kms / max(klaunch, 1)
    vals = torch.tensor([ms, kernel_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    ms_max, kernel_ms_max = float(vals[0]), float(vals[1])

    # ---- e2e through the public API: pinned host points in, grid (slab) out ----
    host_pts = torch.from_numpy(w.points).pin_memory()
    host_out = torch.empty(tuple(out.shape), dtype=torch.float32).pin_memory()
    e2e_steps = max(1, min(args.steps, 10))
    barrier()
    eb, ee = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        eb.record(stream)
        for _ in range(e2e_steps):
            dpts = host_pts.to(dev, non_blocking=True)
            if t1 > t0:
                plan.compute_slab(dpts, t0, t1, n_norm=w.n, out=out, stream=stream)
            host_out.copy_(out, non_blocking=True)
        ee.record(stream)
    barrier()
    e2e_ms = torch.tensor([eb.elapsed_time(ee) / e2e_steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_ms = float(e2e_ms.item())
    h2d = w.points.nbytes * world
    d2h = w.G[0] * w.G[1] * w.G[2] * 4

    # ---- roofline of the dominant kernel (the tile kernel) ----
    (hbm_peak, hbm_src), (bf16_peak, bf16_src) = peaks()
    grid_bytes = w.G[0] * w.G[1] * (t1 - t0) * 4
    t_fp32 = 2.0 * C / (FP32_NOMINAL_TFLOPS * 1e12)
    t_hbm = grid_bytes / (hbm_peak * 1e9)
    if t_fp32 >= t_hbm:
        ach = 2.0 * C / (kernel_ms * 1e-3) / 1e12
        roof = {"bound": "alu", "achieved": ach, "peak": FP32_NOMINAL_TFLOPS, "unit": "TFLOP/s",
                "frac": ach / FP32_NOMINAL_TFLOPS,
                "peak_source": "derived: 148 SMs x 128 FP32 lanes x 2 FLOP x 1.965 GHz (DESIGN.md §4); "
                               "tools/fma_peak measured 74.2 TFLOP/s FFMA2"}
    else:
        ach = grid_bytes / (kernel_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak,
                "peak_source": hbm_src}
    roof["traffic"] = profile_traffic(w.name, info["engine"])
    roof["kernel"] = KERNELS[info["engine"]] % info["Bt"]
    roof["kernel_ms"] = kernel_ms_max
    roof["algorithmic"] = {"flops": 2 * C, "bytes": grid_bytes,
                           "per_unit": "2 FLOP per contribution (one FMA acc += K_s*K_t), 4 B per voxel written once"}
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
                   "useful_fraction": C / (128 * 32 * mma_cols / args.steps)}

    result = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            m = min(ORACLE_SAMPLE[w.name], w.n)
            Cs, dt = run_oracle_sample(w, m)
            cpu = {"value": Cs / dt, "unit": UNIT, "cores": host_cores(), "kind": "oracle",
                   "sample": "first %d of %d points, full %dx%dx%d grid, FP64 oracle (PB form), %.1f s"
                             % (m, w.n, *w.G, dt)}
        result = {
            "metric": METRIC, "value": C_total / (ms_max * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_dict(w, info, {"contributions": C_total, "ms_per_grid": ms_max,
                                            "parallelism": "time-slab x%d" % world, "slab_cuts": cuts,
                                            "l2": "flushed between timed steps (256 MiB write, untimed)",
                                            "inputs_resident": True}),
            "e2e": {"value": C_total / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms},
            "gpu_launches": own * args.steps,
            "library_launches": {"cub_calls": cub * args.steps},
            "clocks": clk.summary(),
            "roofline": roof,
            "roofline_tensor": roof_tc,
            "engine": ENGINES[info["engine"]],
            "cpu_baseline": cpu,
        }
        print(json.dumps(result))
    plan.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def profile_traffic(name, engine):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the tile kernel from the
    committed ncu --set full capture of this workload and engine (profiles/traffic.json)."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        try:
            return json.load(open(p)).get("%s/engine%d" % (name, engine))
        except Exception:
            return None
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="stress", choices=sorted(CONFIG_INDEX))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and rank == 0:
        print("warning: --gpus %d but WORLD_SIZE %d" % (args.gpus, world), file=sys.stderr)
    w = synth.make_config(args.config)
    if args.impl == "reference":
        return reference_main(args, w, rank)
    return gpu_main(args, w, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
