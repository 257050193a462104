#!/bin/bash
# Profiles for profiles/ (run on the GPU box from the repo root, after the same
# commands exited 0 without ncu):
#   launch list (gpu__time_duration.sum, clock-control none) of the default bench,
#   ncu --set full of one step's k_mc launches (the dominant kernel), and of
#   k_pairs<1> and k_integrate.  Usage: scripts/profile_round.sh [CONFIG]
set -x
C=${1:-C1}
O=gpurun_out/prof
mkdir -p $O
B="python bench.py --config $C --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file $O/${C}_launches.csv $B > $O/${C}_launches.log 2>&1
NMC=$(grep -c -E '::k_mc<|::k_approx<' $O/${C}_launches.csv)
NMC=$((NMC / 2))   # launches per step (warm-up + timed step)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_mc|k_approx' \
  --launch-skip $NMC -c $NMC -o $O/${C}_kmc -f $B > $O/${C}_kmc.log 2>&1
NK=$(grep -c -E '::k_pairs|::k_integrate' $O/${C}_launches.csv)
NK=$((NK / 2))
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_pairs|k_integrate' \
  --launch-skip $NK -c $NK -o $O/${C}_k1comb -f $B > $O/${C}_k1comb.log 2>&1
ls -la $O
