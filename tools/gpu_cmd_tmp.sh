timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 900 python tools/c4_sweep.py c4 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('refine_s', round(d['refine_s'],2), 'beta_min', d['beta_min']); print([ (round(x['beta'],3), x['waves'], x['relaxations'], round(x['kernel_ms'],1)) for x in d['single']]); print(d['batched_sweep'])"
timeout 600 python tools/bench_search.py c1 c2 c3 --reps 3 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['config'], d['beta'], d['status'], d['relaxations'], d['kernel_ms'], round(d['edges_relaxed_per_s']/1e9,3))"
timeout 300 python tools/bench_build.py 64 3 > gpurun_out/bb.log 2>&1; python -c "import json; d=json.loads(open('gpurun_out/bb.log').read().strip().splitlines()[-1]); print(d['lib'], {k: round(v,2) for k,v in d['kernel_ms'].items()})"
