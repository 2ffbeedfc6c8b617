python -m pytest tests/test_reset_ahead_gpu.py tests/test_parity_gpu.py tests/test_rollout_gpu.py -x -q 2>&1 | tail -3
timeout 300 python tools/time_prebuild.py c3 2>&1 | tail -1
timeout 300 python tools/steady.py c3 100 200 2>&1 | tail -1
XMG_AHEAD=0 timeout 300 python tools/steady.py c3 100 200 2>&1 | tail -1
timeout 300 python tools/prof_rollout.py c3 100 32 2 1 2>&1 | tail -2
