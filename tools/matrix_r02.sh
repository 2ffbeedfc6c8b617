python -m pytest tests/test_reset_ahead_gpu.py tests/test_parity_gpu.py tests/test_registry_gpu.py -x -q 2>&1 | tail -1
for w in c3 c4 doorkey; do timeout 300 python tools/time_prebuild.py $w 2>&1 | tail -1; done
timeout 300 python tools/steady.py c3 100 200 | tail -1
