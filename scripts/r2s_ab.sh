#!/bin/bash
O=gpurun_out/${1:-r2s}
mkdir -p $O
for C in ${CONFIGS:-C4}; do
  for V in ${MODES:-3 1 2 0}; do
    NLFEM_COMB_OVERLAP=$V timeout 900 python bench.py --config $C --steps ${STEPS:-1} --warmup 1 --no-e2e --no-cpu-baseline > $O/ov${V}_$C.json 2> $O/ov${V}_$C.err
    python -c "
import json; d=json.load(open('$O/ov${V}_$C.json')); r=d['roofline']; p=d['phase_ms']
print('overlap=$V %-4s'%'$C', 'ms/step %.2f'%d['ms_per_step'], 'pairs %.1f integ %.1f units %.1f rest %.1f'%(p[1],p[3],p[5],p[3]-p[5]), 'frac %.3f'%r['frac'])"
  done
done
