for k in 1 2 3 4c5; do timeout -s KILL 300 python tools/precond_cmp.py $k 1 > gpurun_out/s16_$k.log 2>&1; tail -3 gpurun_out/s16_$k.log; done
