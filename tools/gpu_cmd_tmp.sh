for v in b1 b2; do MPAP_LIB=paper_1705_02408_b200/libmpap_$v.so timeout 300 python tools/bench_build.py 64 3 2>&1 | tail -1 | cut -c1-400; done
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
