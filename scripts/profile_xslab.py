"""One x-slab of a config (slab k of N cost-balanced cuts) computed a few times, for ncu launch
lists of a rank's step (development aid).  usage: profile_xslab.py CONFIG N K"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1705_09366_b200 as S  # noqa: E402
import stkde_synth as synth  # noqa: E402

name, N, K = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
w = synth.make_config(name)
dev = torch.device("cuda", 0)
t = torch.from_numpy(w.points).to(dev)
with S.Plan(max_n=w.n, device=0, **w.grid_kwargs()) as p:
    cuts = p.xslab_partition(t, N)
    a, b = cuts[K], cuts[K + 1]
    out = torch.empty((b - a, w.G[1], w.G[2]), device=dev)
    for _ in range(3):
        p.compute_xslab(t, a, b, n_norm=w.n, out=out)
    torch.cuda.synchronize()
    print("slab", a, b)
