"""Run the tcgen05 engine on (a prefix of) a config; prints ok (development aid)."""
import os
import sys

os.environ.setdefault("STKDE_ENGINE", "2")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1705_09366_b200 as S  # noqa: E402
import stkde_synth as synth  # noqa: E402

name, m = sys.argv[1], int(sys.argv[2])
w = synth.make_config(name)
pts = w.points[:m]
dev = torch.device("cuda", 0)
t = torch.from_numpy(pts).to(dev)
with S.Plan(max_n=len(pts), device=0, **w.grid_kwargs()) as p:
    out = p.compute(t)
    torch.cuda.synchronize()
    print("ok", name, m, p.info()["chunk_candidates"], flush=True)
