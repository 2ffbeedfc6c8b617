#!/bin/bash
# ncu --set full of one reset-ahead batch (prebuild_kernel) at C3: the batch of epoch 16.
python tools/prof_step.py c3 20 1 > gpurun_out/prof_pre_plain.log 2>&1 || { echo plain_failed; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prebuild -c 1 \
  -o gpurun_out/r02_c3_prebuild python tools/prof_step.py c3 20 1 > gpurun_out/ncu_pre.log 2>&1; echo pre_rc=$?
