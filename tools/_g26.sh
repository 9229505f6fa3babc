timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
OPT=9 VALUES=1,0 timeout 300 python tools/ab_options.py 2>&1 | tail -2
