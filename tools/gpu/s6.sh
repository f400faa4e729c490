timeout 300 python tools/prof_tm.py 4 1 3 2>&1 | tail -1
timeout 300 python tools/prof_tm.py 4 1 3 0 2>&1 | tail -1
timeout 300 python tools/prof_tm.py 4 8 3 2>&1 | tail -1
timeout 300 python tools/prof_tm.py 5 1 3 2>&1 | tail -1
timeout 300 python tools/prof_tm.py 2 4 3 2>&1 | tail -1
timeout 300 python tools/prof_tm.py 3 16 3 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_solve.py tests/test_gpu_loopback.py -q -x --timeout=900 -p no:cacheprovider -k "not config3" 2>&1 | tail -3
