#!/bin/bash
# Round-2 profile session (run under gpurun): launch list + ncu --set full of
# the step kernels at C3 steady state (step 100) and across the budget-reset
# burst (steps 505-507).  Every ncu command runs only after the same command
# exited 0 without ncu.
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none"
python tools/prof_step.py c3 505 3 > gpurun_out/prof_plain.log 2>&1 || { echo plain_failed; exit 1; }
timeout 600 ncu $M -c 1100 --csv --log-file gpurun_out/r02_launches_c3.csv python tools/prof_step.py c3 505 3 \
  > gpurun_out/ncu_l.log 2>&1; echo launches_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_ -s 201 -c 2 \
  -o gpurun_out/r02_c3_steady python tools/prof_step.py c3 100 3 > gpurun_out/ncu_full.log 2>&1; echo steady_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_ -s 1011 -c 4 \
  -o gpurun_out/r02_c3_burst python tools/prof_step.py c3 505 3 > gpurun_out/ncu_burst.log 2>&1; echo burst_rc=$?
