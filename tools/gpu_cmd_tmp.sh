timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench6.json 2> gpurun_out/bench6.err; echo bench=$? >> gpurun_out/res.txt
timeout 600 python tools/bench_search.py c1 c2 c3 c4 --reps 3 > gpurun_out/search6.jsonl 2>&1
timeout 900 python tools/c4_sweep.py c4 > gpurun_out/c4sweep6.json 2>&1
