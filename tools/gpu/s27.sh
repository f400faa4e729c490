# SM-bound or memory-bound diagnostic, refreshed workloads beyond the bench (config 5 apply, weak line, config 3)
timeout -s KILL 300 python tools/prof_l2.py 801 33 187 0 > gpurun_out/s27_l2.log 2>&1
timeout -s KILL 300 python tools/prof_l2.py 801 99 61 0 >> gpurun_out/s27_l2.log 2>&1
cat gpurun_out/s27_l2.log
timeout -s KILL 400 python tools/prof_tm.py 5 1 3 > gpurun_out/s27_cfg5_apply.log 2>&1; tail -1 gpurun_out/s27_cfg5_apply.log
timeout -s KILL 600 python bench.py --weak --steps 5 --warmup 3 > gpurun_out/s27_weak.json 2> gpurun_out/s27_weak.err; echo weak=$?; tail -c 1500 gpurun_out/s27_weak.json
timeout -s KILL 900 python bench.py --config 3 --no-cpu-baseline --no-e2e > gpurun_out/s27_cfg3.json 2> gpurun_out/s27_cfg3.err; echo cfg3=$?; tail -c 600 gpurun_out/s27_cfg3.err
