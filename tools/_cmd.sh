timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in "2 4 300" "3 16 60"; do echo -n "solve $c: "; timeout 300 python tools/solve_iter.py $c 2>&1 | tail -1; done
for z in 6 12 17 34; do echo -n "ZC=$z solve 2 4: "; HZ_CP_ZC=$z timeout 300 python tools/solve_iter.py 2 4 300 2>&1 | tail -1 | cut -c1-150; done
for c in "2 4 c64" "2 1 c64" "4 1 c64" "3 16 c64" "5 1 c64"; do echo -n "apply $c: "; timeout 300 python tools/prof_apply.py $c 2>&1 | tail -1 | cut -c1-220; done
