timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_solve.py -x -q 2>&1 | tail -2
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print({k:d[k] for k in ['value','ms_per_step','iterations','relres_max','apply_kernel_gpts_s','apply_share_of_step','e2e']}, d['roofline']['frac'])"
