"""Run small parity cases / configs on the watchdog (DIAG) build and report the first
mbarrier wait that timed out (development aid).  usage: tc_watch_case.py NAME[:ENV=V,..] ..."""
import os
import sys

os.environ["STKDE_TC_WATCHDOG"] = "1"
os.environ.setdefault("STKDE_LIB_PATH", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                     "paper_1705_09366_b200", "libstkde_prof.so"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch  # noqa: E402

import paper_1705_09366_b200 as S  # noqa: E402
import stkde_synth as synth  # noqa: E402

TAGS = {6: "ld:empty0", 7: "ld:empty1", 8: "ld:recbar", 9: "gen:full", 10: "gen:done0", 11: "gen:done1",
        12: "gen:dempty(mma)", 13: "gen:dempty(handover)", 14: "epi:dfull"}
for arg in sys.argv[1:]:
    name, _, envs = arg.partition(":")
    for kv in filter(None, envs.split(",")):
        k, v = kv.split("=")
        os.environ[k] = v
    if name in synth.CONFIGS:
        w = synth.make_config(name)
        pts, g, kid = w.points, w.grid_kwargs(), 0
    else:
        import test_gpu_parity as T
        case = [c for c in T.SMALL if c[0] == name][0]
        _, n, g, kid, cl = case
        pts = T.make_points(n, g, cl, seed=len(name))
    dev = torch.device("cuda", 0)
    t = torch.from_numpy(pts).to(dev)
    with S.Plan(max_n=len(pts), device=0, kernel=kid, **g) as p:
        out = p.compute(t)
        torch.cuda.synchronize()
        rec = p.tc_profile()[31]
        info = p.info()
        if rec:
            tag = (rec >> 48) & 0x7FFF
            print("%s %s: WATCHDOG tag=%d (%s) block=%d warp=%d parity=%d" % (
                name, envs, tag, TAGS.get(tag, "?"), (rec >> 24) & 0xFFFFFF, (rec >> 8) & 0xFFFF, rec & 0xFF), flush=True)
        else:
            print("%s %s: no watchdog event, Bt=%d sum=%g" % (name, envs, info["Bt"], float(out.double().sum())), flush=True)
    for kv in filter(None, envs.split(",")):
        os.environ.pop(kv.split("=")[0])
