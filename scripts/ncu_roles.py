"""ncu SASS source page + nvdisasm line table -> per-role / per-line instruction and stall
summary of the tcgen05 tile kernel (development aid).
usage: ncu_roles.py <sass csv> <nvdisasm -g -c dump> <function substring> [top]"""
import collections
import csv
import re
import sys

ncu_csv, dis, fun = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
SRC = "/root/repo/paper_1705_09366_b200/csrc/stkde_tile_tc.cu"
src = open(SRC).read().split("\n")
ld_lo = next(i for i, l in enumerate(src, 1) if "=== LOADER ===" in l)
gen_lo = next(i for i, l in enumerate(src, 1) if "=== GENERATORS ===" in l)
ep_lo = next(i for i, l in enumerate(src, 1) if "epilogue: D -> registers" in l)
kern_lo = next(i for i, l in enumerate(src, 1) if "k_tile_tc(const GridParams g" in l)

line_of, infun, pend, last = {}, False, [], -1
for ln in open(dis):
    if ln.startswith("//--------------------- .text."):
        infun = fun in ln
        continue
    if not infun:
        continue
    m = re.match(r'\s*//## File "([^"]+)", line (\d+)', ln)
    if m:
        pend.append((m.group(1).split("/")[-1], int(m.group(2))))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m:
        if pend:
            # outermost line inside the kernel body of stkde_tile_tc.cu
            cands = [l for f, l in pend if f == "stkde_tile_tc.cu" and l >= kern_lo]
            last = cands[-1] if cands else ([l for f, l in pend if f == "stkde_tile_tc.cu"] or [-1])[-1]
            pend = []
        line_of[int(m.group(1), 16)] = last

rows = list(csv.reader(open(ncu_csv)))
hdr, data = rows[1], rows[2:]
ia, ie = hdr.index("Address"), hdr.index("Instructions Executed")
samp = hdr.index("Warp Stall Sampling (All Samples)")
scols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
base = int(data[0][ia], 16)
per_line = collections.defaultdict(lambda: [0, 0, collections.Counter()])
for r in data:
    l = line_of.get(int(r[ia], 16) - base, -1)
    a = per_line[l]
    a[0] += int(r[ie] or 0)
    a[1] += int(r[samp] or 0)
    for h in scols:
        v = int(r[hdr.index(h)] or 0)
        if v:
            a[2][h[6:]] += v
TI = sum(a[0] for a in per_line.values()) or 1
TS = sum(a[1] for a in per_line.values()) or 1


def role(l):
    if l < kern_lo:
        return "helpers/other"
    if l < ld_lo:
        return "setup"
    if l < gen_lo:
        return "loader"
    if l < ep_lo:
        return "gen k-block"
    return "epilogue+tail"


agg = collections.defaultdict(lambda: [0, 0, collections.Counter()])
for l, (i, s_, st) in per_line.items():
    a = agg[role(l)]
    a[0] += i
    a[1] += s_
    a[2].update(st)
print("total inst %.3e  samples %d" % (TI, TS))
for k, (i, s_, st) in sorted(agg.items(), key=lambda x: -x[1][1]):
    tot = sum(st.values()) or 1
    print("  %-14s inst %5.1f%%  samples %5.1f%%   %s" % (k, 100 * i / TI, 100 * s_ / TS,
          ", ".join("%s %d%%" % (n, 100 * v / tot) for n, v in st.most_common(5))))
print()
for l, (i, s_, st) in sorted(per_line.items(), key=lambda x: -x[1][1])[:top]:
    tot = sum(st.values()) or 1
    txt = src[l - 1].strip()[:70] if l > 0 else ""
    print("%5.1f%%s %5.1f%%i %5d [%-13s] %-34s %s" % (100 * s_ / TS, 100 * i / TI, l, role(l),
          ",".join("%s%d" % (n, 100 * v / tot) for n, v in st.most_common(3)), txt))
