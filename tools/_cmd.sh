timeout 120 python tools/prof_apply.py 3 1 c64 5 > /dev/null || { echo "TMA TEST FAILED/HUNG rc=$?"; exit 1; }
timeout 120 python tools/diag_decomp.py 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in "4 1 c64" "5 1 c64" "3 1 c64" "2 1 c64" "2 4 c64"; do timeout 300 python tools/prof_apply.py $c | cut -c1-160; done
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-large | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print({k:d[k] for k in ['value','ms_per_step','iterations','relres_max','apply_kernel_gpts_s','apply_share_of_step']}, d['roofline']['frac'])"
