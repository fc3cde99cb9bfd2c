"""Phase profile of the tcgen05 tile kernel (development aid): STKDE_TC_PROF=1."""
import os
import sys

os.environ["STKDE_TC_PROF"] = "1"
os.environ.setdefault("STKDE_LIB_PATH", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1705_09366_b200", "libstkde_prof.so"))
os.environ.setdefault("STKDE_ENGINE", "2")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1705_09366_b200 as S  # noqa: E402
import stkde_synth as synth  # noqa: E402

GEN = ["wait_full", "tables+bar1", "stage_wait", "S_gen", "K_gen", "wait_st+bar2", "mma_issue", "epilogue",
       "kblocks", "after_batch", "total"]
LD = ["segments", "cand_rounds", "wait_empty", "sort", "scatter+chords", "kbinfo+publish", "batches", "total",
      "wait_tma"]
for name in sys.argv[1:] or ["stress"]:
    w = synth.make_config(name)
    dev = torch.device("cuda", 0)
    t = torch.from_numpy(w.points).to(dev)
    with S.Plan(max_n=w.n, device=0, **w.grid_kwargs()) as p:
        out = torch.empty(w.G, device=dev)
        p.compute(t, out=out)
        p.tc_profile()
        p.compute(t, out=out)
        v = p.tc_profile()
        gt, lt = v[10] or 1, v[23] or 1
        print("%s: generators (sum over teams, cycles): %s" % (name, ", ".join(
            "%s %.1f%%" % (n, 100.0 * (v[i] + (v[11] + v[12] + v[13] + v[14] if i == 7 else 0) + (v[15] if i == 6 else 0)) / gt)
            for i, n in enumerate(GEN[:8]))))
        print("    k-blocks %d, per k-block per team %.0f cycles" % (v[8], v[10] / max(v[8], 1) * 1.0))
        print("%s: loader: %s, batches %d" % (name, ", ".join(
            "%s %.1f%%" % (n, 100.0 * v[16 + i] / lt) for i, n in list(enumerate(LD))[:6] + [(8, "wait_tma")]),
            v[22]))
        if os.environ.get("STKDE_MMALAT"):
            print("    MMA commit->complete latency (issuing lane spins): %.0f cycles per k-block" % (v[14] / max(v[8], 1)))
        print("    mma_issue split: fence+setup %.1f%%, mma+commit+sync %.1f%% (of generator cycles)" % (
            100.0 * v[15] / gt, 100.0 * v[6] / gt))
        print("    epilogue: wait+sync %.1f%%, tmem ld+cvt %.1f%%, bulk read wait %.1f%%, stage+issue %.1f%%, tail %.1f%%"
              % tuple(100.0 * v[i] / gt for i in (11, 12, 14, 13, 7)))
        print("    stage waits > 200 cycles: %d of %d k-blocks (%d at a batch's first k-block)" % (
            v[9] >> 40, v[8], (v[9] >> 20) & 0xFFFFF))
