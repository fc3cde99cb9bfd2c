"""Time the adaptive-bandwidth pass (stkde_compute_adaptive) per config -- development aid."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1705_09366_b200 as S  # noqa: E402
import stkde_synth as synth  # noqa: E402

dev = torch.device("cuda", 0)
for name in sys.argv[1:] or ["stress"]:
    w = synth.make_config(name)
    t = torch.from_numpy(w.points).to(dev)
    bw = torch.from_numpy(synth.adaptive_bandwidths(w)).to(dev)
    with S.Plan(max_n=w.n, device=0, **w.grid_kwargs()) as p:
        out = torch.empty(w.G, device=dev)
        for _ in range(3):
            p.compute_adaptive(t, bw, out=out)
        torch.cuda.synchronize()
        p.enable_kernel_timing(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            p.compute_adaptive(t, bw, out=out)
        e1.record()
        torch.cuda.synchronize()
        kms, kl = p.kernel_ms()
        print("%-7s adaptive step %.3f ms  tile %.3f ms" % (name, e0.elapsed_time(e1) / 10, kms / max(kl, 1)), flush=True)
