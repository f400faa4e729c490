# launch list of BiCGSTAB and BiCGStab(2) iterations on config 4 (2 RHS): kernel shares of the solve leg
timeout 600 python tools/prof_solve.py 10 1 2 > gpurun_out/s31_solve1.log 2>&1; tail -1 gpurun_out/s31_solve1.log | cut -c1-80
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/s31_solve_ell1_launches.csv python tools/prof_solve.py 10 1 2 > gpurun_out/s31_ncu1.log 2>&1; echo ncu1=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/s31_solve_ell2_launches.csv python tools/prof_solve.py 10 2 2 > gpurun_out/s31_ncu2.log 2>&1; echo ncu2=$?
