#!/bin/bash
# ncu --set full + source counters of one launch of a kernel; summary, raw and
# per-line stall tables written on the box.
#   scripts/profile_kernel.sh TAG KERNEL_REGEX CONFIG SKIP
T=${1:-prof}
K=${2:-k_integrate}
C=${3:-C3n}
SKIP=${4:-5}
O=gpurun_out/$T
mkdir -p $O
B="python bench.py --config $C --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"$K" --launch-skip $SKIP -c 1 \
  -o /tmp/${T} -f $B > $O/ncu.log 2>&1
python scripts/ncu_summary.py /tmp/${T}.ncu-rep > $O/summary.txt 2>&1
python scripts/ncu_lines.py /tmp/${T}.ncu-rep "$K" 0 60 > $O/lines.txt 2>&1
ncu -i /tmp/${T}.ncu-rep --page source --csv > $O/source.csv 2> $O/source.err
ncu -i /tmp/${T}.ncu-rep --page raw --csv > $O/raw.csv 2> $O/raw.err
ls -la $O
