#!/bin/bash
# quick k_mc measurement on the GPU box: C1 and P3f bench lines (no e2e / CPU
# baseline) plus the fullcaps parity tests.  Usage: scripts/quick_perf.sh TAG
T=${1:-q}
O=gpurun_out/$T
mkdir -p $O
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize_values.py -m gpu -x -q -s \
  -k "fullcaps or C1 or C4 or C3f or oracle" -p no:cacheprovider > $O/tests.log 2>&1
echo "tests_rc=$?" >> $O/tests.log
for C in ${CONFIGS:-C1 P3f}; do
  python bench.py --config $C --steps ${STEPS:-5} --warmup 3 --no-e2e --no-cpu-baseline \
    > $O/$C.json 2> $O/$C.err
done
tail -3 $O/tests.log
for C in ${CONFIGS:-C1 P3f}; do python -c "
import json,sys; d=json.load(open('$O/$C.json')); r=d['roofline']
print('$C', 'ms/step %.2f'%d['ms_per_step'], 'units ms %.2f'%r['launch_ms'], 'frac %.3f'%r['frac'], 'phases', d['phase_ms'])"; done
