# ncu --set full of the solve iteration's kernels on config 4 (2 RHS): bicg_update, bicg_s, the DOT4 apply
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bicg_update -s 3 -c 1 -o gpurun_out/r02_bicg_update_cfg4 python tools/prof_solve.py 6 1 2 > gpurun_out/s32_a.log 2>&1; echo a=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bicg_s_kernel -s 3 -c 1 -o gpurun_out/r02_bicg_s_cfg4 python tools/prof_solve.py 6 1 2 > gpurun_out/s32_b.log 2>&1; echo b=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:apply27_tm -s 7 -c 1 -o gpurun_out/r02_apply27_tm_dot4_cfg4 python tools/prof_solve.py 6 1 2 > gpurun_out/s32_c.log 2>&1; echo c=$?
ls -la gpurun_out/*.ncu-rep
