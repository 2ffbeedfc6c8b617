#!/bin/bash
# Launch lists (time + DRAM bytes per launch) of the step kernels for the
# non-default workloads, merged into profiles/ncu_summary.json, then the bench
# line of each workload (which reads its traffic from that summary).  Every
# ncu command runs only after the same command exited 0 without ncu.
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none"
wls=${*:-"c1 c2 doorkey c4"}
for wl in $wls; do
  python tools/prof_step.py $wl 100 3 > gpurun_out/prof_plain_$wl.log 2>&1 && \
    timeout 600 ncu $M -s 200 -c 12 --csv --log-file gpurun_out/launches_$wl.csv python tools/prof_step.py $wl 100 3 \
    > gpurun_out/ncu_l_$wl.log 2>&1
  echo "launches $wl rc=$?"
done
python tools/ncu_workloads.py r01 $wls > gpurun_out/ncu_workloads.log 2>&1; echo "merge rc=$?"
for wl in $wls; do
  timeout 900 python bench.py --workload $wl > gpurun_out/bench_$wl.json 2> gpurun_out/bench_$wl.err
  echo "bench $wl rc=$?"
done
