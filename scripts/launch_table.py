"""Per-kernel totals from an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    m = re.search(r"(k_[a-z_0-9]+(<[a-z0-9, ]+>)?|at::[a-z_:]+)", r[ki])
    name = m.group(1) if m else r[ki][:30]
    scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
             "second": 1e3, "s": 1e3}[r[ui]]
    tot[name] += float(r[vi].replace(",", "")) * scale
    cnt[name] += 1
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 1
T = sum(tot.values())
print(f"{'kernel':28s} {'launches':>8s} {'ms/run':>10s} {'share':>7s}   (runs={runs}, total {T / runs:.3f} ms/run)")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:28s} {cnt[k]:8d} {v / runs:10.3f} {v / T * 100:6.1f}%")
