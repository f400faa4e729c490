timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in "2 4 300" "3 16 60"; do echo -n "solve $c: "; timeout 300 python tools/solve_iter.py $c 2>&1 | tail -1; done
for c in "2 4 c64" "4 1 c64" "3 16 c64" "5 1 c64"; do echo -n "apply $c: "; timeout 300 python tools/prof_apply.py $c 2>&1 | tail -1 | cut -c1-220; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:apply27_cp -c 2 -o gpurun_out/cp7_solve python tools/solve_iter.py 2 4 3 > gpurun_out/cp_ncu_solve.log 2>&1; tail -1 gpurun_out/cp_ncu_solve.log
