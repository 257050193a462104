"""Sum dram__bytes_read.sum + dram__bytes_write.sum (and durations) over the
kernels of an ncu report whose name matches a regex.

usage: ncu_traffic.py REPORT [REGEX]"""
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
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0,
         "msecond": 1e-3, "second": 1.0}


def val(row, name):
    i = H.index(name)
    return float(row[i].replace(",", "")) * scale.get(U[i], 1.0)


tot_b = tot_t = 0.0
for r in rows[2:]:
    name = r[H.index("Kernel Name")].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
    if not pat.search(name):
        continue
    b = val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
    t = val(r, "gpu__time_duration.sum")
    tot_b += b
    tot_t += t
    print(f"{name:28s} dram {b / 1e6:10.2f} MB  {t * 1e6:9.1f} us  {b / t / 1e9:8.1f} GB/s")
print(f"{'total':28s} dram {tot_b / 1e6:10.2f} MB  {tot_t * 1e6:9.1f} us  "
      f"{tot_b / max(tot_t, 1e-30) / 1e9:8.1f} GB/s  bytes={int(tot_b)}")
