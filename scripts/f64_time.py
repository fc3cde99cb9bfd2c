"""FP64-output option timing (stkde_compute_f64, CUDA events, inputs resident).
usage: python scripts/f64_time.py <config>..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1705_09366_b200 as S  # noqa: E402
import stkde_synth as synth  # noqa: E402

for name in sys.argv[1:]:
    w = synth.make_config(name); g = w.grid_kwargs()
    with S.Plan(max_n=w.n, device=0, **g) as p:
        t = torch.from_numpy(w.points).cuda()
        out = p.compute_f64(t)
        for _ in range(2): p.compute_f64(t, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); k = 3
        for _ in range(k): p.compute_f64(t, out=out)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / k
        C = int(p.count_contributions(t).item())
        print("%s f64: %.3f ms, %.3e contributions/s" % (name, ms, C / ms * 1e3))
