"""Key metrics of one kernel in an ncu --set full report -> JSON (profiles/ summaries).
usage: ncu_summary.py <report.ncu-rep> <out.json> [note]"""
import csv
import io
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
note = sys.argv[3] if len(sys.argv) > 3 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
        "launch__block_size", "launch__registers_per_thread", "sm__cycles_active.avg",
        "sm__inst_executed.avg.per_cycle_active", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active"]
d = {}
for k in KEYS:
    if k in hdr:
        i = hdr.index(k)
        d[k] = (vals[i] + " " + units[i]).strip()
st = {}
for i, h in enumerate(hdr):
    if h.startswith("smsp__average_warp_latency_issue_stalled_") or h.startswith("smsp__average_warps_issue_stalled_"):
        name = h.split("stalled_")[1].split(".")[0].split("_per_")[0]
        try:
            st[name] = st.get(name, 0.0) + float(vals[i].replace(",", ""))
        except ValueError:
            pass
tot = sum(v for k, v in st.items() if k not in ("selected",)) or 1.0
if st:
    s_all = sum(st.values()) or 1.0
    d["stall_share_pct"] = {k: round(100 * v / s_all, 1) for k, v in sorted(st.items(), key=lambda x: -x[1])[:10]}
def _bytes(v):
    num, unit = v.split()[0].replace(",", ""), (v.split() + [""])[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
    return float(num) * scale


try:
    d["dram_bytes_total"] = int(_bytes(d["dram__bytes_read.sum"]) + _bytes(d["dram__bytes_write.sum"]))
except Exception:
    pass
d["_kernel"] = note
json.dump(d, open(out, "w"), indent=1)
print(json.dumps(d, indent=1))
