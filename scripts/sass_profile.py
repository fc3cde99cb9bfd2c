"""Summarise an ncu --page source --csv --print-source sass dump: instruction mix,
stall reasons and the hottest source-level regions (development aid)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
ie = hdr.index("Instructions Executed")
samp = hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[ie] or 0) for r in data)
ts = sum(int(r[samp] or 0) for r in data)
cnt, smp = collections.Counter(), collections.Counter()
for r in data:
    op = r[1].split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    o = o.split(".")[0]
    cnt[o] += int(r[ie] or 0)
    smp[o] += int(r[samp] or 0)
print("total inst %.3e, samples %d" % (tot, ts))
print("  " + ", ".join("%s %.1f%%(s%.1f%%)" % (o, 100 * c / tot, 100 * smp[o] / ts) for o, c in cnt.most_common(16)))
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tots = {h: sum(int(r[hdr.index(h)] or 0) for r in data) for h in cols}
s = sum(tots.values())
print("  stalls: " + ", ".join("%s %.1f%%" % (h[6:], 100 * v / s) for h, v in sorted(tots.items(), key=lambda x: -x[1])[:8]))
# contiguous regions by address: bucket into windows of 64 instructions
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
win = 48
regions = []
for i in range(0, len(data), win):
    chunk = data[i:i + win]
    regions.append((sum(int(r[samp] or 0) for r in chunk), sum(int(r[ie] or 0) for r in chunk), i, chunk))
for sm, ins, i, chunk in sorted(regions, key=lambda x: -x[0])[:n]:
    ops = collections.Counter((r[1].split()[1] if r[1].split()[0].startswith("@") else r[1].split()[0]).split(".")[0]
                              for r in chunk if r[1].split())
    print("  region %5d: samples %5.1f%% inst %5.1f%%  %s" % (i, 100 * sm / ts, 100 * ins / tot,
                                                            ",".join("%s%d" % kv for kv in ops.most_common(6))))
