set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q --timeout=900 -p no:cacheprovider > gpurun_out/s1_pytest.log 2>&1; echo pytest=$?
tail -30 gpurun_out/s1_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/s1_bench.json 2> gpurun_out/s1_bench.err; echo bench=$?
cat gpurun_out/s1_bench.json | head -c 600
