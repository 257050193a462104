#!/bin/bash
# every bench workload once (GPU box, repo root) -> gpurun_out/bench/<config>.json
mkdir -p gpurun_out/bench
for c in ${CFGS:-C0 C1 C1n C1a C2 C3n C3f C4}; do
  st=5; [ $c = C4 ] && st=3; [ $c = C3f ] && st=3; [ $c = C2 ] && st=3
  timeout 1200 python bench.py --config $c --steps $st --warmup 3 > gpurun_out/bench/$c.json 2> gpurun_out/bench/$c.err
  echo "$c rc=$?"
done
