#!/bin/bash
# One GPU measurement session (run under gpurun): tests, smoke, the driver's
# bench commands, the other configs' bench lines, ncu launch lists and
# --set full captures.  Every ncu command runs only after the same command
# exited 0 without ncu.  Outputs in gpurun_out/ (tools/make_profiles.py <tag>
# copies the summaries into profiles/).
T=${1:-r02}
G=gpurun_out
python __graft_entry__.py > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $G/${T}_pytest_gpu.log 2>&1; echo pytest_rc=$?
timeout 600 python __graft_entry__.py smoke > $G/${T}_smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python bench.py --steps 20 --warmup 5 > $G/${T}_bench_c3_k20.json 2> $G/${T}_bench_c3_k20.err; echo bench20_rc=$?
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $G/${T}_bench_ref_k20.json 2> $G/${T}_bench_ref_k20.err; echo ref20_rc=$?
timeout 900 python bench.py > $G/${T}_bench_c3.json 2> $G/${T}_bench_c3.err; echo bench_rc=$?
for wl in c2 c4 doorkey; do
  timeout 900 python bench.py --workload $wl --steps 256 --warmup 5 --no-image > $G/${T}_bench_$wl.json 2> $G/${T}_bench_$wl.err; echo bench_${wl}_rc=$?
done
for wl in c1 c2; do
  timeout 900 python bench.py --workload $wl --steps 256 --warmup 5 --no-image --graph > $G/${T}_bench_${wl}_graph.json 2> $G/${T}_bench_${wl}_graph.err; echo bench_${wl}_graph_rc=$?
done
timeout 900 python bench.py --workload c1 --steps 256 --warmup 5 --no-image > $G/${T}_bench_c1.json 2> $G/${T}_bench_c1.err; echo bench_c1_rc=$?
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none"
# the driver's command: launch list over its timed window (the kernels after the reset and the
# 496 untimed steps: split_batch, policy keys, actions, reset, 496 x 3 step kernels + 31 batches)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 1520 -c 120 --csv \
  --log-file $G/${T}_launches_bench_c3_k20.csv python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu \
  --no-fused --no-block --no-image --no-windows > $G/${T}_ncu_bench.log 2>&1; echo launches_bench_rc=$?
for wl in c3 c4 doorkey c2 c1; do
  python tools/prof_step.py $wl 100 3 > /dev/null 2>&1 && \
    timeout 600 ncu $M -s 200 -c 12 --csv --log-file $G/launches_$wl.csv python tools/prof_step.py $wl 100 3 \
    > $G/ncu_l_$wl.log 2>&1
  echo launches_${wl}_rc=$?
done
python tools/prof_step.py c3 505 3 > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:step_ -s 201 -c 2 -o $G/${T}_c3_steady python tools/prof_step.py c3 100 3 > $G/ncu_full.log 2>&1; echo full_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_main -s 505 -c 2 \
  -o $G/${T}_c3_burst python tools/prof_step.py c3 505 3 > $G/ncu_burst.log 2>&1; echo burst_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prebuild -c 1 \
  -o $G/${T}_c3_prebuild python tools/prof_step.py c3 20 1 > $G/ncu_pre.log 2>&1; echo pre_rc=$?
python tools/prof_rollout.py c3 100 32 2 1 > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none \
  --import-source on -k regex:rollout -s 1 -c 1 -o $G/${T}_c3_rollout python tools/prof_rollout.py c3 100 32 2 1 \
  > $G/ncu_roll.log 2>&1; echo roll_rc=$?
python tools/prof_image.py 16384 5 2 > /dev/null 2>&1 && timeout 300 ncu --set full --clock-control none \
  --import-source on -k regex:image_kernel -s 1 -c 1 -o $G/${T}_image python tools/prof_image.py 16384 5 1 \
  > $G/ncu_img.log 2>&1; echo img_rc=$?
