#!/bin/bash
# full -m gpu suite, then bench lines (phases) for the default build and the
# round-start library (old) side by side.   scripts/r2g_run.sh TAG
O=gpurun_out/${1:-r2g}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/tests.log 2>&1
echo "tests_rc=$?" >> $O/tests.log
tail -3 $O/tests.log
NOTEST=1 LIBS="${LIBS:-default old}" CONFIGS="${CONFIGS:-C1 C3n C3f C2}" bash scripts/r2e_ab.sh ${1:-r2g}
