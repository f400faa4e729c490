# config-4 solve iteration breakdown: timing, then the ncu launch list of 20 iterations
timeout -s KILL 300 python tools/prof_solve.py 20 1 2 > gpurun_out/s21_time.log 2>&1
timeout -s KILL 300 python tools/prof_solve.py 20 2 2 >> gpurun_out/s21_time.log 2>&1
cat gpurun_out/s21_time.log
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/s21_launches.csv python tools/prof_solve.py 20 1 2 > gpurun_out/s21_ncu.log 2>&1
echo ncu rc=$?
