#!/bin/bash
# Round-2 (session 3) GPU run: full -m gpu suite with the Philox4x32-7 stream,
# the C4 headline bench line, and K1 occupancy variants timed by phase.
O=gpurun_out/r2c
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/tests.log 2>&1
echo "tests_rc=$?" >> $O/tests.log
tail -3 $O/tests.log
timeout 600 python bench.py --steps 3 --warmup 3 > $O/C4.json 2> $O/C4.err
python -c "
import json; d=json.load(open('$O/C4.json')); r=d['roofline']
print('C4', 'ms/step %.1f'%d['ms_per_step'], 'value %.3g'%d['value'], 'e2e %.3g'%d['e2e']['value'], 'frac %.3f'%r['frac'], 'phases', d.get('phase_ms'))"
for L in default k4 k5; do
  for C in C2 C3n; do
    if [ $L = default ]; then unset NLFEM_GPU_LIB; else export NLFEM_GPU_LIB=$PWD/paper_2302_07499_b200/libnlfem_gpu_$L.so; fi
    timeout 600 python bench.py --config $C --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/${L}_$C.json 2> $O/${L}_$C.err
    python -c "
import json; d=json.load(open('$O/${L}_$C.json')); r=d['roofline']
print('$L $C', 'ms/step %.2f'%d['ms_per_step'], 'frac %.3f'%r['frac'], 'phases', d.get('phase_ms'))"
  done
done
