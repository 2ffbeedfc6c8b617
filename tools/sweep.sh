#!/bin/bash
# C5 (BASELINE.json configs[4]): num_envs sweep 2^10..2^24 on one GPU for
# DoorKey-8x8 and XLand-R4-13x13 medium, through bench.py (timed window with
# the budget reset burst; kernel legs off).  Output: gpurun_out/sweep.jsonl
out=gpurun_out/sweep.jsonl
: > $out
for wl in doorkey c3; do
  for p in 10 12 14 16 18 20 22 24; do
    n=$((1 << p))
    timeout 600 python bench.py --workload $wl --envs $n --steps 512 --warmup 4 --no-e2e --no-cpu \
      --no-image 2>> gpurun_out/sweep.err | tail -1 >> $out
    echo "$wl 2^$p rc=$?"
  done
done
