for a in "4 1 3" "4 1 3 0" "4 8 3" "2 4 3"; do timeout 300 python tools/prof_tm.py $a 2>&1 | tail -1; done
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "random or baseline or tiled or edges" 2>&1 | tail -1
timeout -s KILL 120 python tools/dbg_solve.py 1 1 2>&1 | tail -2
