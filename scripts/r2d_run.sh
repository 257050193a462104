#!/bin/bash
# Round-2 (session 4) GPU run: smoke, the full -m gpu suite and the C4 headline
# bench line with the code as committed.
O=gpurun_out/r2d
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke_rc=$?" >> $O/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/tests.log 2>&1
echo "tests_rc=$?" >> $O/tests.log
tail -3 $O/tests.log
timeout 600 python bench.py --steps 3 --warmup 3 > $O/C4.json 2> $O/C4.err
python -c "
import json; d=json.load(open('$O/C4.json')); r=d['roofline']
print('C4', 'ms/step %.1f'%d['ms_per_step'], 'value %.3g'%d['value'], 'e2e %.3g'%d['e2e']['value'], 'frac %.3f'%r['frac'], 'phases', d.get('phase_ms'))"
for C in C1 C2 C3n C3f; do
  timeout 600 python bench.py --config $C --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/$C.json 2> $O/$C.err
  python -c "
import json; d=json.load(open('$O/$C.json')); r=d['roofline']
print('$C', 'ms/step %.2f'%d['ms_per_step'], 'frac %.3f'%r['frac'], 'phases', d.get('phase_ms'))"
done
