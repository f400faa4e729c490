timeout 600 ncu --set full --clock-control none --import-source on -k regex:apply27_tm -s 2 -c 1 -o gpurun_out/s5_tm_cfg4 python tools/prof_tm.py 4 1 3 > gpurun_out/s5_ncu.log 2>&1; echo ncu=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:apply27_tm -s 2 -c 1 -o gpurun_out/s5_tm_cfg4_8 python tools/prof_tm.py 4 8 3 > gpurun_out/s5_ncu8.log 2>&1; echo ncu=$?
