#!/bin/bash
# overlap mode (combine of chunk k beside the units of chunk k+1) on / off
O=gpurun_out/${1:-r2o}
mkdir -p $O
[ -z "$NOTEST" ] && { timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize_values.py tests/test_gpu_chunks.py tests/test_gpu_distributed.py tests/test_gpu_checked.py -x -q -p no:cacheprovider > $O/tests.log 2>&1; echo "tests_rc=$?" >> $O/tests.log; tail -2 $O/tests.log; }
for C in ${CONFIGS:-C3f C2 C1}; do
  for V in 1 0; do
    NLFEM_COMB_OVERLAP=$V timeout 900 python bench.py --config $C --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > $O/ov${V}_$C.json 2> $O/ov${V}_$C.err
    python -c "
import json; d=json.load(open('$O/ov${V}_$C.json')); r=d['roofline']; p=d['phase_ms']
print('overlap=$V %-4s'%'$C', 'ms/step %.2f'%d['ms_per_step'], 'pairs %.1f integ %.1f units %.1f rest %.1f'%(p[1],p[3],p[5],p[3]-p[5]), 'frac %.3f'%r['frac'])"
  done
done
