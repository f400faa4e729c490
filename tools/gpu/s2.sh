set -x

timeout 300 python tools/prof_tm.py 4 1 3 2>&1 | tail -2
timeout 300 python tools/prof_tm.py 4 8 3 2>&1 | tail -2
timeout 300 python tools/prof_tm.py 2 1 3 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout=600 -p no:cacheprovider 2>&1 | tail -15
