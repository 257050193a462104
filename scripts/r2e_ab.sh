#!/bin/bash
# Combine (k_integrate) A/B on the GPU box: parity tests with the default
# build, then bench lines per library variant with the phase times
# (integration - units = the combine's share of the step).  scripts/r2e_ab.sh TAG
O=gpurun_out/${1:-r2e}
mkdir -p $O
[ -z "$NOTEST" ] && timeout 1800 python -m pytest ${TESTS:-tests/test_gpu_parity.py tests/test_gpu_fullsize_values.py tests/test_gpu_chunks.py tests/test_gpu_distributed.py} \
  -x -q -p no:cacheprovider > $O/tests.log 2>&1
echo "tests_rc=$?" >> $O/tests.log
tail -2 $O/tests.log
for C in ${CONFIGS:-C3n C3f}; do
  for L in ${LIBS:-default old}; do
    if [ $L = default ]; then unset NLFEM_GPU_LIB; else export NLFEM_GPU_LIB=$PWD/paper_2302_07499_b200/libnlfem_gpu_$L.so; fi
    timeout 900 python bench.py --config $C --steps ${STEPS:-3} --warmup ${WARM:-3} --no-e2e --no-cpu-baseline \
      > $O/${L}_$C.json 2> $O/${L}_$C.err
    python -c "
import json; d=json.load(open('$O/${L}_$C.json')); r=d['roofline']; p=d['phase_ms']
print('%-8s %-4s'%('$L','$C'), 'ms/step %.2f'%d['ms_per_step'], 'pairs %.1f pattern %.1f integ %.1f units %.1f combine %.1f'%(p[1],p[2],p[3],p[5],p[3]-p[5]), 'frac %.3f'%r['frac'])"
  done
done
