#!/bin/bash
# Round-2 full check on the GPU box: the -m gpu suite, smoke, the C4 headline
# bench line (e2e + CPU baseline), quick lines for the other configs, and the
# C4 profiles.   scripts/r2_full.sh TAG
O=gpurun_out/${1:-full}
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -x -q -s -p no:cacheprovider > $O/tests.log 2>&1
echo "tests_rc=$?" >> $O/tests.log
tail -2 $O/tests.log
timeout 1200 python bench.py > $O/C4.json 2> $O/C4.err
for C in ${CONFIGS:-C1 C3n P3f}; do
  timeout 900 python bench.py --config $C --steps 3 --warmup 3 --no-e2e --no-cpu-baseline \
    > $O/$C.json 2> $O/$C.err
done
for C in C4 ${CONFIGS:-C1 C3n P3f}; do python -c "
import json; d=json.load(open('$O/$C.json')); r=d['roofline']
print('$C', 'ms/step %.2f'%d['ms_per_step'], 'units ms %.2f'%r['launch_ms'], 'frac %.3f'%r['frac'], 'phases', d['phase_ms'], 'e2e', (d.get('e2e') or {}).get('value'))"; done
[ -n "$PROF" ] && bash scripts/profile_c4.sh ${1:-full}_prof
ls $O
