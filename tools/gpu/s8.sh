timeout -s KILL 280 python tools/dbg_solve.py 1 1 > gpurun_out/s8.log 2>&1; echo rc=$? >> gpurun_out/s8.log
