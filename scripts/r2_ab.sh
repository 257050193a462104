#!/bin/bash
# Round-2 A/B run on the GPU box: correctness of the default build, k_mc
# moment variants timed side by side (NLFEM_GPU_LIB), fixed-point precision,
# owner-computes emulation.   scripts/r2_ab.sh TAG
O=gpurun_out/${1:-ab}
mkdir -p $O
[ -z "$NOTEST" ] && timeout 1800 python -m pytest ${TESTS:-tests/test_gpu_parity.py tests/test_gpu_fullsize_values.py tests/test_gpu_distributed.py} \
  -x -q -s -p no:cacheprovider > $O/tests.log 2>&1
echo "tests_rc=$?" >> $O/tests.log
tail -2 $O/tests.log
for L in ${LIBS:-default m0 m1 m2}; do
  for C in ${CONFIGS:-C1 P3f C2}; do
    if [ $L = default ]; then unset NLFEM_GPU_LIB; else export NLFEM_GPU_LIB=$PWD/paper_2302_07499_b200/libnlfem_gpu_$L.so; fi
    timeout 900 python bench.py --config $C --steps ${STEPS:-3} --warmup ${WARM:-3} --no-e2e --no-cpu-baseline \
      > $O/${L}_$C.json 2> $O/${L}_$C.err
    python -c "
import json; d=json.load(open('$O/${L}_$C.json')); r=d['roofline']
print('$L $C', 'ms/step %.2f'%d['ms_per_step'], 'units ms %.2f'%r['launch_ms'], 'frac %.3f'%r['frac'], 'hits', d['mc_hits'])"
  done
done
unset NLFEM_GPU_LIB
[ -n "$PREC" ] && timeout 900 python scripts/fixed_point_precision.py $PREC > $O/precision.json 2> $O/precision.err
[ -n "$EMU" ] && for C in $EMU; do timeout 1500 python scripts/owner_computes_emulate.py ${C%:*} ${C#*:} > $O/emulate_${C%:*}.jsonl 2> $O/emulate_${C%:*}.err; done
ls $O
