# final verification of the round: GPU suite, the default bench line, its launch list
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s28_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/s28_tests.log
timeout 1200 python bench.py > gpurun_out/s28_bench.json 2> gpurun_out/s28_bench.err; echo bench=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s28_ref.json 2> gpurun_out/s28_ref.err; echo ref=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s28_launches.csv python bench.py --steps 2 --warmup 1 --no-solve --no-extra --no-cpu-baseline > gpurun_out/s28_ncu_l.log 2>&1; echo ncu1=$?
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s28_smoke.log 2>&1; echo smoke=$?; tail -2 gpurun_out/s28_smoke.log
