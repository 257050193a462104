"""Summarise an ncu report: key metrics and stall reasons per kernel."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
idi = h.index("ID")
want = ["Duration", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "L1/TEX Hit Rate", "L2 Hit Rate", "Warp Cycles Per Issued Instruction",
        "Avg. Active Threads Per Warp", "Branch Efficiency", "Waves Per SM"]
seen = set()
for r in rows[1:]:
    k = r[idi] + " " + r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "")[:24]
    if r[mi] in want and (k, r[mi]) not in seen:
        seen.add((k, r[mi]))
        print(f"{k:30s} {r[mi]:40s} {r[vi]:>12s} {r[ui]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
H = rr[0]
for row in rr[2:]:
    name = row[H.index("Kernel Name")].split("(")[0].replace("void ", "").replace("<unnamed>::", "")[:24]
    st = {}
    for i, col in enumerate(H):
        if col.startswith("smsp__pcsamp_warps_issue_stalled_") and not col.endswith("not_issued"):
            try:
                st[col.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(row[i].replace(",", ""))
            except ValueError:
                pass
    tot = sum(st.values()) or 1
    top = sorted(st.items(), key=lambda x: -x[1])[:6]
    print(name, " | ".join(f"{k} {v / tot * 100:.0f}%" for k, v in top))
    for col in ("sm__sass_thread_inst_executed_op_dfma_pred_on.sum", "sm__sass_thread_inst_executed_op_dadd_pred_on.sum",
                "sm__sass_thread_inst_executed_op_dmul_pred_on.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
                "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
                "smsp__inst_executed.sum", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
                "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"):
        if col in H:
            print("   ", col, row[H.index(col)], rr[1][H.index(col)])
