"""Executed FP64 work per kernel of an ncu --set full report: thread-level
DFMA / DADD / DMUL instructions per elapsed cycle (FLOPs = 2 DFMA + DADD +
DMUL, summed over the SMs), times the SM clock -- the executed counterpart of
bench.py's ledger FLOPs.

usage: ncu_fp64.py REPORT [REGEX]"""
import csv
import re
import subprocess
import sys

rep = sys.argv[1]
pat = re.compile(sys.argv[2] if len(sys.argv) > 2 else ".")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(raw.splitlines()))
H, U = rows[0], rows[1]
scale = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9,
         "us": 1e-6, "ms": 1e-3, "s": 1.0}


def col(name):
    for i, h in enumerate(H):
        if h == name:
            return i
    return None


def num(r, name):
    i = col(name)
    return float(r[i].replace(",", "")) if i is not None and r[i] else 0.0


clk = 1.965e9  # SM clock during the capture (--clock-control none, 1965 MHz)
tot_f = tot_t = 0.0
for r in rows[2:]:
    kname = r[H.index("Kernel Name")].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
    if not pat.search(kname):
        continue
    fma2 = num(r, "derived__smsp__sass_thread_inst_executed_op_dfma_pred_on_x2")
    add = num(r, "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed")
    mul = num(r, "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed")
    it = col("gpu__time_duration.sum")
    t = float(r[it].replace(",", "")) * scale.get(U[it], 1.0)
    rate = (fma2 + add + mul) * clk  # FLOP/s
    tot_f += rate * t
    tot_t += t
    print(f"{kname:28s} per cycle: 2xDFMA {fma2:7.0f} DADD {add:7.0f} DMUL {mul:7.0f} -> "
          f"{rate / 1e12:6.2f} TFLOP/s executed over {t * 1e6:8.1f} us")
print(f"{'total':28s} {tot_f:.3e} FLOP executed in {tot_t * 1e6:.1f} us = "
      f"{tot_f / max(tot_t, 1e-30) / 1e12:.2f} TFLOP/s")
