python -m pytest tests/test_reset_ahead_gpu.py tests/test_rollout_gpu.py -x -q 2>&1 | tail -2
for a in 1 0; do
XMG_AHEAD=$a timeout 300 python tools/prof_rollout.py c3 100 32 4 1 2>&1 | tail -1
XMG_AHEAD=$a timeout 300 python tools/prof_rollout.py c3 100 32 4 0 2>&1 | tail -1
XMG_AHEAD=$a timeout 300 python tools/prof_rollout.py c3 490 32 2 1 2>&1 | tail -1
done
