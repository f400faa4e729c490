set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -k host_buffers -x -q --timeout=300 2>&1 | tail -3
timeout 600 python bench.py --no-solve --no-extra > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err; echo rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 1 --no-solve --no-extra --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:apply27_tm -c 1 -o gpurun_out/r2_apply27_tm_cfg4_nrhs8 python bench.py --steps 1 --warmup 1 --no-solve --no-extra --no-e2e --no-cpu-baseline > gpurun_out/ncu_f8.log 2>&1; echo ncu2=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:apply27_tm -c 1 -o gpurun_out/r2_apply27_tm_cfg4_nrhs1 python tools/prof_tm.py 4 1 1 > gpurun_out/ncu_f1.log 2>&1; echo ncu3=$?
