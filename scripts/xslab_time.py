"""Time one full-width x-slab compute (stkde_compute_xslab over [0, Gx)) per config -- with
STKDE_PLAIN_STORES=1 this is the direct gather's store path on one GPU (development aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1705_09366_b200 as S  # noqa: E402
import stkde_synth as synth  # noqa: E402

dev = torch.device("cuda", 0)
for name in sys.argv[1:] or ["social", "stress"]:
    w = synth.make_config(name)
    t = torch.from_numpy(w.points).to(dev)
    with S.Plan(max_n=w.n, device=0, **w.grid_kwargs()) as p:
        out = torch.empty(w.G, device=dev)
        for _ in range(3):
            p.compute_xslab(t, 0, w.G[0], out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            p.compute_xslab(t, 0, w.G[0], out=out)
        e1.record()
        torch.cuda.synchronize()
        print("%-7s plain=%s  x-slab pass %.3f ms" % (name, os.environ.get("STKDE_PLAIN_STORES", "0"),
                                                     e0.elapsed_time(e1) / 10), flush=True)
