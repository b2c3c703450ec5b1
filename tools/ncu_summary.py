"""Summarise an ncu --set full report of k_eval_fused (reads the .ncu-rep with the ncu CLI)."""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
d = {h: (vals[i], units[i]) for i, h in enumerate(hdr)}


SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6, "second": 1e3}


def num(k, to_base=False):
    try:
        v = float(d[k][0])
    except Exception:
        return None
    if to_base:
        v *= SCALE.get(d[k][1], 1.0)
    return v


out = {
    "kernel": d.get("Kernel Name", ("?",))[0],
    "gpu__time_duration_ms": num("gpu__time_duration.sum", True),
    "dram_bytes_read": num("dram__bytes_read.sum", True),
    "dram_bytes_write": num("dram__bytes_write.sum", True),
    "dmma_pipe_active_pct": num("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active"),
    "tensor_pipe_realtime_pct_elapsed": num("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"),
    "fp64_pipe_pct": num("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
    "lsu_pipe_pct": num("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
    "shared_wavefronts_pct": num("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
    "shared_bank_conflicts_ld": num("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"),
    "shared_bank_conflicts_st": num("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum"),
    "registers_per_thread": num("launch__registers_per_thread"),
    "issue_active_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "sm_clock_ghz": num("gpc__cycles_elapsed.avg.per_second"),
}
if out["dram_bytes_read"] is not None:
    out["dram_bytes_per_launch"] = out["dram_bytes_read"] + (out["dram_bytes_write"] or 0)
stalls = {}
for h, (v, u) in d.items():
    if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
        try:
            stalls[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v)
        except ValueError:
            pass
tot = sum(stalls.values()) or 1.0
out["stall_share"] = {k: round(v / tot, 4) for k, v in sorted(stalls.items(), key=lambda x: -x[1]) if v / tot > 0.005}
if len(sys.argv) > 2:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(src)))
    sh = srows[1]
    ix = {h: i for i, h in enumerate(sh)}
    data = srows[2:]
    key = "Warp Stall Sampling (All Samples)"
    tot = sum(float(r[ix[key]] or 0) for r in data)
    top = sorted(data, key=lambda r: -float(r[ix[key]] or 0))[:int(sys.argv[2])]
    out["top_sass"] = [(r[ix["Address"]][-5:], round(float(r[ix[key]]) / tot, 4), r[ix["Source"]].strip()) for r in top]
print(json.dumps(out, indent=1))
