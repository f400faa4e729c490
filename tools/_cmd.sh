timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
for c in "4 1 c64" "4 4 c64"; do timeout 300 python tools/prof_apply.py $c | cut -c1-300; done
HZ_CFG5_NZ=401 timeout 600 python tools/prof_apply.py 5 1 c64 10 | cut -c1-300
