#!/bin/bash
# ncu --set full of one chunk's k_mc launches (chunk 51 of the C4 step: 8
# launches, the two streams' lists) and of the K1 / combine launches of the same
# step region; summaries written on the box, reports deleted.
#   scripts/profile_c4.sh [TAG] [SKIP_KMC] [CONFIG]
T=${1:-c4prof}
SKIP=${2:-400}
C=${3:-C4}
O=gpurun_out/$T
mkdir -p $O
B="python bench.py --config $C --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 1500 ncu --set full --clock-control none -k regex:k_mc --launch-skip $SKIP -c 8 \
  -o /tmp/${T}_kmc -f $B > $O/kmc_ncu.log 2>&1
python scripts/ncu_summary.py /tmp/${T}_kmc.ncu-rep > $O/kmc_summary.txt 2>&1
python scripts/ncu_fp64.py /tmp/${T}_kmc.ncu-rep > $O/kmc_fp64.txt 2>&1
python scripts/ncu_traffic.py /tmp/${T}_kmc.ncu-rep > $O/kmc_traffic.txt 2>&1
timeout 1500 ncu --set full --clock-control none -k regex:'k_pairs|k_integrate' --launch-skip 20 -c 4 \
  -o /tmp/${T}_k1 -f $B > $O/k1_ncu.log 2>&1
python scripts/ncu_summary.py /tmp/${T}_k1.ncu-rep > $O/k1_summary.txt 2>&1
python scripts/ncu_traffic.py /tmp/${T}_k1.ncu-rep > $O/k1_traffic.txt 2>&1
ls -la $O
