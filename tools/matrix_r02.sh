python tools/graph_probe.py c1 2000
python tools/graph_probe.py c2 1000
python tools/graph_probe.py c1 200 > /dev/null && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 400 -c 30 --csv --log-file gpurun_out/c1_graph_launches.csv python tools/graph_probe.py c1 200 > /dev/null 2>&1; echo ncu=$?
