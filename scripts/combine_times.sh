#!/bin/bash
# Pure kernel time of the combine (k_integrate) launches of one step, per
# library variant, from an ncu launch list (serialized, clock-control none).
#   LIBS="default old" scripts/combine_times.sh TAG CONFIG
T=${1:-ct}
C=${2:-C3n}
O=gpurun_out/$T
mkdir -p $O
for L in ${LIBS:-default old}; do
  if [ $L = default ]; then unset NLFEM_GPU_LIB; else export NLFEM_GPU_LIB=$PWD/paper_2302_07499_b200/libnlfem_gpu_$L.so; fi
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"${KERN:-k_integrate}" -c 5000 --csv \
    --log-file $O/${L}_$C.csv python bench.py --config $C --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $O/${L}_$C.log 2>&1
  python - <<PY
import csv
tot={}; n={}
for r in csv.reader(open('$O/${L}_$C.csv')):
    if len(r)>5 and r[-1].replace('.','').replace(',','').isdigit() and 'gpu__time_duration' in r[-3]:
        k=r[4].split('(')[0][-40:]; u=r[-2]; v=float(r[-1].replace(',',''))
        v*= {'ns':1e-6,'us':1e-3,'ms':1,'s':1e3}.get(u,1e-6)
        tot[k]=tot.get(k,0)+v; n[k]=n.get(k,0)+1
for k in tot: print('$L $C', k, 'launches', n[k], 'total ms %.2f'%tot[k])
PY
done
