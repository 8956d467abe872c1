MPAP_DEBUG_TIMING=1 timeout 300 python tools/bench_build.py 64 2 2>&1 | tail -30 | cut -c1-300
