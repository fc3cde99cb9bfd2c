"""Quick per-config timing of stkde_compute (CUDA events) -- development aid."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1705_09366_b200 as S  # noqa: E402
import stkde_synth as synth  # noqa: E402

names = sys.argv[1:] or ["tiny", "dengue", "social", "ornith", "stress"]
dev = torch.device("cuda", 0)
for name in names:
    w = synth.make_config(name)
    g = w.grid_kwargs()
    t = torch.from_numpy(w.points).to(dev)
    with S.Plan(max_n=w.n, device=0, **g) as p:
        out = torch.empty(w.G, device=dev)
        C = int(p.count_contributions(t).item())
        for _ in range(3):
            p.compute(t, out=out)
        torch.cuda.synchronize()
        p.enable_kernel_timing(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        K = 10
        e0.record()
        for _ in range(K):
            p.compute(t, out=out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / K
        kms, kl = p.kernel_ms()
        info = p.info()
        gr = p.graph(t, out=out)                     # the same call as one CUDA graph per step
        for _ in range(3):
            gr.launch()
        e0.record()
        for _ in range(K):
            gr.launch()
        e1.record()
        torch.cuda.synchronize()
        gms = e0.elapsed_time(e1) / K
        gr.close()
        p.check()
        print("%-7s n=%-8d C=%.3e  step %.3f ms  graph %.4f ms  tile kernel %.3f ms  -> %.3e contrib/s  tile=%dx%dx%d CT=%d occ=%d chunk=%d launches=%d+%dcub eng=%d"
              % (name, w.n, C, ms, gms, kms / max(kl, 1), C / (ms * 1e-3), info["Bx"], info["By"], info["Bt"],
                 info["tile_layers_per_thread"], info["tile_ctas_per_sm"], info["chunk_candidates"],
                 info["last_own_launches"], info["last_cub_calls"], info["engine"]), flush=True)
