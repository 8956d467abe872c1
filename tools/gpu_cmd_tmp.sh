timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 600 python tools/bench_search.py c1 --reps 3 2>&1 | tail -4
