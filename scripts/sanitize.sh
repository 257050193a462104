#!/bin/bash
# compute-sanitizer evidence (one tool per gpurun call):
#   scripts/sanitize.sh memcheck|racecheck|synccheck|initcheck
# runs the smoke assembly and a C1 fullcaps step forced into many chunks
# (NLFEM_PAIRS_PER_CHUNK: two alternating unit-buffer sets, four streams).
T=${1:-memcheck}
O=gpurun_out/san
mkdir -p $O
CS="compute-sanitizer --tool $T --error-exitcode 9 --print-limit 50"
[ "$T" = memcheck ] && CS="$CS --leak-check no"
timeout 1200 $CS python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1
echo "smoke rc=$?" >> $O/${T}_smoke.log
NLFEM_PAIRS_PER_CHUNK=${CHUNK:-300000} timeout 2400 $CS python bench.py --config ${CFG:-C1} \
  --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/${T}_c1chunks.log 2>&1
echo "c1chunks rc=$?" >> $O/${T}_c1chunks.log
tail -3 $O/${T}_smoke.log $O/${T}_c1chunks.log
