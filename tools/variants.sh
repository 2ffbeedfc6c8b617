#!/bin/bash
# Compare libxmg builds (XMG_LIB) on bench.py's timed window.
# usage: tools/variants.sh "<workloads>" lib1.so lib2.so ...
wls=$1; shift
for L in "$@"; do
  for wl in $wls; do
    XMG_LIB=$L timeout 600 python bench.py --workload $wl --steps 512 --warmup 4 --no-e2e --no-cpu --no-fused \
      --no-image 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$L', '$wl', 'value %.4e step_ms %.4f main_ms %.4f rare_ms %.4f frac %.3f' % (d['value'], d['ms_per_step'], r['kernel_ms'], r['rare_kernel_ms'], r['frac']))"
  done
done
