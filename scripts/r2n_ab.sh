#!/bin/bash
# co-residency experiment: units launches capped at 3 CTAs/SM by shared-memory
# padding (NLFEM_MC_PAD_KB) with 128-thread combine CTAs beside them
O=gpurun_out/${1:-r2n}
mkdir -p $O
run() { # tag lib pad config
  if [ $2 = default ]; then unset NLFEM_GPU_LIB; else export NLFEM_GPU_LIB=$PWD/paper_2302_07499_b200/libnlfem_gpu_$2.so; fi
  if [ $3 = 0 ]; then unset NLFEM_MC_PAD_KB; else export NLFEM_MC_PAD_KB=$3; fi
  timeout 900 python bench.py --config $4 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > $O/$1_$4.json 2> $O/$1_$4.err
  python -c "
import json; d=json.load(open('$O/$1_$4.json')); r=d['roofline']; p=d['phase_ms']
print('%-14s %-4s'%('$1','$4'), 'ms/step %.2f'%d['ms_per_step'], 'pairs %.1f integ %.1f units %.1f combine %.1f'%(p[1],p[3],p[5],p[3]-p[5]), 'frac %.3f'%r['frac'])"
}
for C in ${CONFIGS:-C3f C2}; do
  run base default 0 $C
  run pad57 default 57 $C
  run ct128 ct128 0 $C
  run ct128pad57 ct128 57 $C
  run ct128pad76 ct128 76 $C
done
