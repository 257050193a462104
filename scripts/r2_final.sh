#!/bin/bash
# Round-2 results on the GPU box: every bench workload once (e2e + CPU
# baseline), the reference arm for C1 / C4, and the ncu launch list of one C4
# step (clock-control none, per-launch durations).   scripts/r2_final.sh TAG
O=gpurun_out/${1:-final}
mkdir -p $O
for c in ${CFGS:-C0 C1 C1n C1a C2 C3n C3f C4}; do
  st=5; [ $c = C4 ] && st=3; [ $c = C3f ] && st=3; [ $c = C2 ] && st=3
  timeout 1500 python bench.py --config $c --steps $st --warmup 3 > $O/$c.json 2> $O/$c.err
  echo "$c rc=$?"
done
for c in C1 C4; do
  timeout 900 python bench.py --impl reference --config $c --steps 2 --warmup 1 > $O/ref_$c.json 2> $O/ref_$c.err
  echo "ref $c rc=$?"
done
[ -n "$LAUNCHES" ] && timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none -c 50000 --csv \
  --log-file $O/C4_launches.csv python bench.py --config C4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline \
  > $O/C4_launches.log 2>&1
[ -f $O/C4_launches.csv ] && python scripts/launch_table.py $O/C4_launches.csv > $O/C4_launch_table.txt 2>&1
ls $O
