timeout 600 ncu --set full --clock-control none --import-source on -k regex:apply27_tm -s 2 -c 1 -o gpurun_out/s3_tm_cfg4 python tools/prof_tm.py 4 1 3 > gpurun_out/s3_ncu.log 2>&1; echo ncu=$?
tail -3 gpurun_out/s3_ncu.log
