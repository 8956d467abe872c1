timeout 300 python tools/bench_build.py 64 3 > gpurun_out/bb.log 2>&1; tail -5 gpurun_out/bb.log | cut -c1-400
