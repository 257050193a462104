"""Top source lines by warp-stall samples for one kernel of an ncu report.

usage: ncu_lines.py REPORT KERNEL_REGEX [LAUNCH_SKIP] [TOP]
"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--launch-skip", skip, "--launch-count", "1", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, rows, tot = "?", [], 0
for r in csv.reader(out.splitlines()):
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif len(r) > 8 and r[0] not in ("", "Line No") and r[2] == "-":
        try:
            s, ins = int(r[4]), int(r[7])
        except ValueError:
            continue
        tot += s
        rows.append((s, ins, fname, r[0], r[1].strip()[:90]))
rows.sort(reverse=True)
print(f"total samples {tot}")
for s, ins, f, ln, src in rows[:top]:
    print(f"{100 * s / max(tot, 1):5.1f}% {ins:>11d} {f}:{ln:<5} {src}")
