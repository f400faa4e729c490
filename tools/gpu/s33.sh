timeout -s KILL 1500 python tools/solve_cfg5.py 25000 > gpurun_out/s33_cfg5_solve.json 2> gpurun_out/s33_cfg5_solve.err; echo rc=$?
cat gpurun_out/s33_cfg5_solve.json; tail -3 gpurun_out/s33_cfg5_solve.err
