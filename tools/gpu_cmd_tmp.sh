timeout 300 python tools/bench_build.py 64 3 2>&1 | grep '"lib"' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['lib'], {k: round(v,1) for k,v in d['kernel_ms'].items()}, d['work']['prefilter_pass'])"
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
