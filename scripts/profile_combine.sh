#!/bin/bash
# ncu --set full (+ source counters) of one combine launch (k_integrate) and the
# source-page CSV, on CONFIG (default C3n).   scripts/profile_combine.sh TAG CONFIG SKIP
T=${1:-comb}
C=${2:-C3n}
SKIP=${3:-5}
O=gpurun_out/$T
mkdir -p $O
B="python bench.py --config $C --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_integrate --launch-skip $SKIP -c 1 \
  -o /tmp/${T}_comb -f $B > $O/comb_ncu.log 2>&1
python scripts/ncu_summary.py /tmp/${T}_comb.ncu-rep > $O/comb_summary.txt 2>&1
ncu -i /tmp/${T}_comb.ncu-rep --page source --csv > $O/comb_source.csv 2> $O/comb_source.err
ncu -i /tmp/${T}_comb.ncu-rep --page raw --csv > $O/comb_raw.csv 2> $O/comb_raw.err
ls -la $O /tmp/${T}_comb.ncu-rep
