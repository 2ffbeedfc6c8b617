#!/bin/bash
# C5 (BASELINE.json configs[4]): num_envs sweep 2^10..2^24 on one GPU for
# DoorKey-8x8 and XLand-R4-13x13 medium-1m, through bench.py (256-step window
# with the budget reset burst; the CPU port on the same envs and window up to
# 2^18 envs).  Output: gpurun_out/<tag>_sweep_c5.jsonl
tag=${1:-r02}
out=gpurun_out/${tag}_sweep_c5.jsonl
: > $out
for wl in doorkey c3; do
  for p in 10 12 14 16 18 20 22 24; do
    n=$((1 << p))
    cpu="--no-cpu"; [ $p -le 18 ] && cpu=""
    timeout 900 python bench.py --workload $wl --envs $n --steps 256 --warmup 4 --no-e2e $cpu --no-image \
      --no-windows 2>> gpurun_out/${tag}_sweep.err | tail -1 >> $out
    echo "$wl 2^$p rc=$?"
  done
done
