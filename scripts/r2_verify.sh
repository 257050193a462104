#!/bin/bash
# Round-2 verification on the GPU box: the whole -m gpu suite, the smoke, and
# quick bench lines (C1, P3f, C4) without e2e / CPU baseline.
O=gpurun_out/${1:-v}
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider -s > $O/tests.log 2>&1
echo "tests_rc=$?" >> $O/tests.log
for C in ${CONFIGS:-C1 P3f C4}; do
  timeout 900 python bench.py --config $C --steps ${STEPS:-3} --warmup 3 --no-e2e --no-cpu-baseline \
    > $O/$C.json 2> $O/$C.err
done
tail -3 $O/smoke.log $O/tests.log
for C in ${CONFIGS:-C1 P3f C4}; do python -c "
import json,sys; d=json.load(open('$O/$C.json')); r=d['roofline']
print('$C', 'ms/step %.2f'%d['ms_per_step'], 'units ms %.2f'%r['launch_ms'], 'frac %.3f'%r['frac'], 'phases', d['phase_ms'])"; done
