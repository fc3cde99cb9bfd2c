"""Run a config with the tcgen05 kernel's mbarrier watchdog on (development aid)."""
import os
import sys

os.environ["STKDE_TC_WATCHDOG"] = "1"
os.environ.setdefault("STKDE_ENGINE", "2")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1705_09366_b200 as S  # noqa: E402
import stkde_synth as synth  # noqa: E402

TAGS = {1: "mma:full", 2: "mma:sfull0", 3: "mma:sfull1", 5: "mma:dfree", 6: "ld:empty0", 7: "ld:empty1",
        8: "ld:recbar", 9: "gen:full", 10: "gen:done0", 11: "gen:done1", 13: "gen:tiledone"}
for name in sys.argv[1:] or ["ornith"]:
    w = synth.make_config(name)
    dev = torch.device("cuda", 0)
    t = torch.from_numpy(w.points).to(dev)
    with S.Plan(max_n=w.n, device=0, **w.grid_kwargs()) as p:
        out = p.compute(t)
        rec = p.tc_profile()[31]
        if rec:
            tag = (rec >> 48) & 0x7FFF
            print("%s: WATCHDOG tag=%d (%s) block=%d warp=%d parity=%d" % (
                name, tag, TAGS.get(tag, "?"), (rec >> 24) & 0xFFFFFF, (rec >> 8) & 0xFFFF, rec & 0xFF))
        else:
            print("%s: no watchdog event" % name)
