python -m pytest tests/test_graph_gpu.py -x -q 2>&1 | tail -1
for e in 32 16 8 4; do XMG_FUSED_EPW=$e python tools/graph_probe.py c1 1000 2>&1 | grep "graph=True" | sed "s/^/epw=$e /"; XMG_FUSED_EPW=$e python tools/graph_probe.py c2 500 2>&1 | grep "graph=True" | sed "s/^/epw=$e /"; done
XMG_FUSED_EPW=4 python -m pytest tests/test_graph_gpu.py -x -q 2>&1 | tail -1
