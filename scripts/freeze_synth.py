"""Write tests/golden/synth_sha256.json: SHA-256 of every config's point array.

Calls only stkde_synth (input plumbing); no oracle or CUDA values are stored.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import stkde_synth as synth  # noqa: E402

out = {"_source": "scripts/freeze_synth.py (stkde_synth generators, SplitMix64 seeds 1-5)"}
for name in synth.CONFIGS:
    w = synth.make_config(name)
    out[name] = {"n": w.n, "sha256": synth.points_sha256(w.points), "G": list(w.G),
                 "hs": w.hs, "ht": w.ht, "sres": w.sres, "tres": w.tres}
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                    "tests", "golden", "synth_sha256.json")
json.dump(out, open(path, "w"), indent=1)
print(path)
