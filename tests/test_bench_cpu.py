"""bench.py's multi-rank control flow on CPU: `--gpus 2` without a torchrun environment
starts 2 ranks itself (torch.distributed.run, gloo in --dry-run), the x-slab cuts come from
the library's host-only partition, and rank 0 alone prints one JSON line."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_self_launches_two_ranks():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "STKDE_BENCH_LAUNCHED")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "1",
                        "--config", "dengue", "--dry-run"], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout                       # rank 0 only
    d = json.loads(lines[0])
    assert d["dry_run"] and d["n_gpus"] == 2 and d["backend"] == "gloo"
    cuts = d["config"]["slab_cuts"]
    assert cuts[0] == 0 and cuts[-1] == 256 and len(cuts) == 3 and all(c % 16 == 0 for c in cuts[:-1])
    assert d["config"]["points_total"] == 11000            # the ranks' slabs partition the points


def test_bench_refuses_mismatched_world():
    # --gpus 2 inside a 1-rank environment is an error, not a silent 1-GPU measurement
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run", "--config", "tiny"],
                       capture_output=True, text=True, env=env, timeout=120)
    assert r.returncode == 2
    assert "error" in json.loads(r.stdout.strip().splitlines()[-1])
