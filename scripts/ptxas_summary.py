"""Registers / spills per kernel from a ptxas -v build log (build.py writes
paper_2302_07499_b200/_build/build.log).  python scripts/ptxas_summary.py [regex]"""
import os
import re
import subprocess
import sys

log = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_2302_07499_b200", "_build", "build.log")
pat = re.compile(sys.argv[1] if len(sys.argv) > 1 else ".")
cur = None
rows = {}
for line in open(log):
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        rows.setdefault(cur, {})["spill"] = (int(m.group(1)), int(m.group(2)))
    m = re.search(r"Used (\d+) registers", line)
    if m:
        rows.setdefault(cur, {})["regs"] = int(m.group(1))
names = list(rows)
dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
for n, d in zip(names, dem):
    short = re.sub(r"\(anonymous namespace\)::", "", d)
    short = re.sub(r"\(.*", "", short)
    if pat.search(short):
        r = rows[n]
        print(f"{short:60s} regs {r.get('regs')}  spill st/ld {r.get('spill')}")
