for L in build_variants/*.so; do XMG_LIB=$L timeout 300 python tools/time_prebuild.py c3 2>&1 | tail -1; done
for L in build_variants/p1g4.so build_variants/p4g4.so; do XMG_LIB=$L timeout 300 python tools/time_prebuild.py c4 2>&1 | tail -1; XMG_LIB=$L timeout 300 python tools/time_prebuild.py doorkey 2>&1 | tail -1; done
