"""Per-phase CUDA-event times of one compute call per config (development aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1705_09366_b200 as S  # noqa: E402
import stkde_synth as synth  # noqa: E402

dev = torch.device("cuda", 0)
for name in sys.argv[1:] or ["tiny", "dengue", "social", "ornith", "stress"]:
    w = synth.make_config(name)
    t = torch.from_numpy(w.points).to(dev)
    with S.Plan(max_n=w.n, device=0, **w.grid_kwargs()) as p:
        out = torch.empty(w.G, device=dev)
        for _ in range(3):
            p.compute(t, out=out)
        p.enable_phase_timing(True)
        K = 10
        for _ in range(K):
            p.compute(t, out=out)
        torch.cuda.synchronize()
        ph, calls = p.phase_ms()
        print("%-7s " % name + "  ".join("%s %.4f" % (k, v / max(calls, 1)) for k, v in ph.items() if v > 0), flush=True)
