XMG_MAIN_P=1 timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_reset_ahead_gpu.py -x -q 2>&1 | tail -2
for p in 0 1; do XMG_MAIN_P=$p timeout 300 python tools/main_probe.py c3 2>&1 | tail -2; XMG_MAIN_P=$p timeout 300 python tools/steady.py c3 100 200 2>&1 | tail -1; done
for p in 0 1; do XMG_MAIN_P=$p timeout 300 python tools/steady.py doorkey 100 200 2>&1 | tail -1; XMG_MAIN_P=$p timeout 300 python tools/steady.py c4 100 200 2>&1 | tail -1; done
