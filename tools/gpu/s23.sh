timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s23_tests.log 2>&1; echo tests=$?
tail -5 gpurun_out/s23_tests.log
timeout 900 python bench.py > gpurun_out/s23_bench.json 2> gpurun_out/s23_bench.err; echo bench=$?
