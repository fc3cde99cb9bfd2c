"""Run stkde_compute on one config a few times (for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1705_09366_b200 as S  # noqa: E402
import stkde_synth as synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "stress"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
w = synth.make_config(name)
dev = torch.device("cuda", 0)
t = torch.from_numpy(w.points).to(dev)
with S.Plan(max_n=w.n, device=0, **w.grid_kwargs()) as p:
    out = torch.empty(w.G, device=dev)
    for _ in range(reps):
        p.compute(t, out=out)
    torch.cuda.synchronize()
    p.check()
print("ok", name, p.info() if False else "")
