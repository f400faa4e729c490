# last check of the committed build: smoke, GPU suite, apply-only bench line
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s34_smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/s34_smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s34_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/s34_tests.log
timeout 600 python bench.py --no-solve --no-extra --no-cpu-baseline > gpurun_out/s34_bench.json 2> gpurun_out/s34_bench.err; echo bench=$?
