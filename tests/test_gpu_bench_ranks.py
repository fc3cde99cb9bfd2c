"""bench.py's N-rank path on a GPU box (rehearsal): `STKDE_BENCH_SHARED_GPU=1 bench.py --gpus 2`
starts 2 torchrun ranks that share the box's GPU(s) round-robin, each computing its cost-balanced
x-slab through the library (graph step, e2e through the public API, the direct IPC gather into
rank 0's grid), with gloo for the bench's own bookkeeping collectives.  Rank 0 alone prints one
line, marked as a rehearsal (its times are not a scaling measurement)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_bench_two_ranks_shared_gpu():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "STKDE_BENCH_LAUNCHED")}
    env["STKDE_BENCH_SHARED_GPU"] = "1"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
                        "--config", "dengue"], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout                       # rank 0 only
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and "rehearsal" in d
    assert d["config"]["parallelism"] == "x-slab x2"
    cuts = d["config"]["slab_cuts"]
    assert cuts[0] == 0 and cuts[-1] == 256 and len(cuts) == 3
    # the ranks' exact per-slab contribution counts add up to the whole grid's C (x-slabs
    # partition the voxels), counted here by one whole-grid call
    import torch

    import paper_1705_09366_b200 as S
    import stkde_synth as synth
    w = synth.make_config("dengue")
    with S.Plan(max_n=w.n, device=0, **w.grid_kwargs()) as p:
        C = int(p.count_contributions(torch.from_numpy(w.points).cuda()).item())
    assert d["config"]["contributions"] == C
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["e2e"]["value"] > 0
    assert d["gpu_launches"] > 0
    direct = d["gather"]["direct"]
    assert "error" not in direct and direct["ms_per_step_into_root"] > 0
