#!/bin/bash
# One GPU session: tests, smoke, bench (+ reference arm), launch lists and ncu
# captures of the step kernels, the fused rollout and the image kernel (run
# under gpurun; every ncu command runs only after the same command exited 0
# without ncu).
set -x
python __graft_entry__.py > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
timeout 600 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none"
python tools/prof_step.py c3 100 3 > gpurun_out/prof_plain.log 2>&1 && \
  timeout 600 ncu $M -s 200 -c 12 --csv --log-file gpurun_out/launches.csv python tools/prof_step.py c3 100 3 \
  > gpurun_out/ncu_l.log 2>&1
echo launches_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_ -s 201 -c 2 \
  -o gpurun_out/prof_c3_full python tools/prof_step.py c3 100 3 > gpurun_out/ncu_full.log 2>&1
echo full_rc=$?
python tools/prof_rollout.py c3 100 32 2 1 > gpurun_out/prof_roll_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:rollout -s 1 -c 1 \
  -o gpurun_out/prof_roll_full python tools/prof_rollout.py c3 100 32 2 1 > gpurun_out/ncu_roll.log 2>&1
echo roll_rc=$?
python tools/prof_image.py 16384 5 2 > gpurun_out/prof_img_plain.log 2>&1 && \
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:image_kernel -s 1 -c 1 \
  -o gpurun_out/prof_image_full python tools/prof_image.py 16384 5 1 > gpurun_out/ncu_img.log 2>&1
echo img_rc=$?
