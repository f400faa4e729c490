# round-2 re-entry check: GPU suite + default bench on HEAD
set -o pipefail
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/s18_pytest.log
echo "pytest rc=$?" >> gpurun_out/s18_pytest.log
timeout -s KILL 600 python bench.py > gpurun_out/s18_bench.json 2> gpurun_out/s18_bench.err
echo "bench rc=$?"
tail -3 gpurun_out/s18_pytest.log
