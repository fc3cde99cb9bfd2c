"""Per-source-line view of an ncu SASS source page (development aid).

usage: ncu_lines.py <ncu --page source --csv --print-source sass dump> <nvdisasm -g -c dump> <function> [top]

Joins ncu's per-instruction samples / executed counts (by offset from the
kernel's first instruction) with nvdisasm's line table of the same cubin and
prints the hottest source lines of stkde_tile_tc.cu with their stall mix."""
import collections
import csv
import re
import sys

ncu_csv, dis, fun = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40

# nvdisasm: offset -> innermost source line
line_of = {}
cur = None
infun = False
for ln in open(dis):
    if ln.startswith("//--------------------- .text."):
        infun = fun in ln
        continue
    if not infun:
        continue
    m = re.match(r'\s*//## File "([^"]+)", line (\d+)', ln)
    if m:
        if "inlined at" not in ln and cur is None or True:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and cur is not None:
        line_of[int(m.group(1), 16)] = cur
        cur_keep = cur

rows = list(csv.reader(open(ncu_csv)))
hdr = rows[1]
data = rows[2:]
ia, ie = hdr.index("Address"), hdr.index("Instructions Executed")
samp = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
base = int(data[0][ia], 16)
agg = collections.defaultdict(lambda: [0, 0, collections.Counter()])
last = None
for r in data:
    off = int(r[ia], 16) - base
    key = line_of.get(off, last)
    last = key
    a = agg[key]
    a[0] += int(r[samp] or 0)
    a[1] += int(r[ie] or 0)
    for h in stall_cols:
        v = int(r[hdr.index(h)] or 0)
        if v:
            a[2][h[6:]] += v
ts = sum(a[0] for a in agg.values()) or 1
ti = sum(a[1] for a in agg.values()) or 1
src = {}
try:
    for i, s in enumerate(open("/root/repo/paper_1705_09366_b200/csrc/stkde_tile_tc.cu"), 1):
        src[i] = s.strip()
except OSError:
    pass
print("samples %d, instructions %.3e" % (ts, ti))
for key, (s, n, st) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    f, l = key if key else ("?", 0)
    stl = ",".join("%s%d" % (k, 100 * v / max(s, 1)) for k, v in st.most_common(3))
    txt = src.get(l, "")[:60] if f == "stkde_tile_tc.cu" else ""
    print("%5.1f%% s  %5.1f%% i  %s:%-4d %-28s %s" % (100 * s / ts, 100 * n / ti, f[:14], l, stl, txt))
