"""Per-phase CUDA-event times of each x-slab of N cost-balanced cuts (development aid):
where a rank's fixed cost goes.  usage: xslab_phases.py CONFIG N"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1705_09366_b200 as S  # noqa: E402
import stkde_synth as synth  # noqa: E402

name, N = sys.argv[1], int(sys.argv[2])
w = synth.make_config(name)
dev = torch.device("cuda", 0)
t = torch.from_numpy(w.points).to(dev)
with S.Plan(max_n=w.n, device=0, **w.grid_kwargs()) as p:
    cuts = p.xslab_partition(t, N)
    for k in range(N):
        a, b = cuts[k], cuts[k + 1]
        out = torch.empty((b - a, w.G[1], w.G[2]), device=dev)
        for _ in range(2):
            p.compute_xslab(t, a, b, n_norm=w.n, out=out)
        torch.cuda.synchronize()
        p.enable_phase_timing(True)
        for _ in range(5):
            p.compute_xslab(t, a, b, n_norm=w.n, out=out)
        ph, calls = p.phase_ms()
        p.enable_phase_timing(False)
        print("%s slab %d [%d, %d): " % (name, k, a, b) + "  ".join("%s %.3f" % (q, v / calls) for q, v in ph.items() if v > 0),
              flush=True)
