"""Time-slab scaling estimate on ONE GPU (development aid): the N cost-balanced slabs of a
config are computed one after another and timed separately; with one rank per GPU and no
collective on the data path, the N-GPU step is the slowest slab, so full / max(slab) is the
ideal N-GPU speedup of the partition (not a multi-GPU measurement)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1705_09366_b200 as S  # noqa: E402
import stkde_synth as synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "stress"
dev = torch.device("cuda", 0)
w = synth.make_config(name)
t = torch.from_numpy(w.points).to(dev)


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


# every step is one CUDA-graph launch (as bench.py times it)
with S.Plan(max_n=w.n, device=0, **w.grid_kwargs()) as p:
    full = torch.empty(w.G, device=dev)
    gfull = p.graph(t, out=full)
    tf = timed(lambda: gfull.launch())
    for kind in ("t", "x"):
        for n in (2, 4, 8):
            cuts = p.slab_partition(t, n) if kind == "t" else p.xslab_partition(t, n)
            ts = []
            for a, b in zip(cuts[:-1], cuts[1:]):
                if kind == "t":
                    gr = p.graph(t, t_begin=a, t_end=b, n_norm=w.n)
                else:
                    gr = p.graph_xslab(t, a, b, n_norm=w.n)
                ts.append(timed(lambda: gr.launch()))
                gr.close()
            print("%s %s-slabs N=%d cuts=%s slab ms=%s -> ideal speedup %.2f (efficiency %.0f %%)" % (
                name, kind, n, cuts, ["%.2f" % x for x in ts], tf / max(ts), 100 * tf / max(ts) / n))
    print("%s full grid %.2f ms" % (name, tf))
