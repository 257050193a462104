#!/bin/bash
# ncu --set full of one step's k_mc launches (the units phase) at CONFIG, with
# the summaries written on the box (the .ncu-rep files are deleted so that
# gpurun_out/ stays small).  Usage: scripts/profile_kmc.sh [CONFIG] [TAG] [REGEX]
C=${1:-P3f}
T=${2:-kmc}
RX=${3:-k_mc}
O=gpurun_out/$T
mkdir -p $O
B="python bench.py --config $C --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file $O/${C}_launches.csv $B > $O/${C}_launches.log 2>&1
N=$(grep -c -E "::$RX" $O/${C}_launches.csv)
N=$((N / 2))
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$RX" \
  --launch-skip $N -c $N -o /tmp/${C}_$T -f $B > $O/${C}_ncu.log 2>&1
ncu -i /tmp/${C}_$T.ncu-rep --page raw --csv > $O/${C}_raw.csv 2>/dev/null
ncu -i /tmp/${C}_$T.ncu-rep --page details --csv > $O/${C}_details.csv 2>/dev/null
python scripts/ncu_summary.py /tmp/${C}_$T.ncu-rep > $O/${C}_summary.txt 2>&1
python scripts/ncu_fp64.py /tmp/${C}_$T.ncu-rep > $O/${C}_fp64.txt 2>&1
ncu -i /tmp/${C}_$T.ncu-rep --page source --csv --print-source sass > $O/${C}_source.csv 2>/dev/null
gzip -f $O/${C}_source.csv $O/${C}_raw.csv
ls -la $O
