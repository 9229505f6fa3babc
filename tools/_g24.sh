timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -2
OPT=9 VALUES=1,0 timeout 300 python tools/ab_options.py 2>&1 | tail -2
