timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r1c_gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r1c_gpu_tests.log
for c in "5 1 c64" "3 1 c64" "2 1 c64"; do timeout 120 python tools/prof_apply.py $c | cut -c1-150; done
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1c_bench.log 2>&1; tail -1 gpurun_out/r1c_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d[k] for k in ['value','ms_per_step','iterations','apply_kernel_gpts_s']}, d['roofline']['frac'], d.get('apply_large'))"
