#!/bin/bash
# Round-2 final run on the GPU box with the committed code: smoke, the full
# -m gpu suite, every bench workload (e2e + CPU baseline), the reference arm at
# C1 / C4, the ncu launch list of one C4 step and the ncu --set full summaries
# of one chunk's k_mc launches and of the K1 / combine launches.
#   scripts/r2m_final.sh TAG
T=${1:-r2m}
O=gpurun_out/$T
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke_rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/tests.log 2>&1
echo "tests_rc=$?" >> $O/tests.log
tail -3 $O/tests.log
LAUNCHES=1 bash scripts/r2_final.sh $T
[ -z "$NOPROF" ] && bash scripts/profile_c4.sh ${T}_prof 400 C4
