timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "c4_golden" 2>&1 | tail -3 >> gpurun_out/res.txt
