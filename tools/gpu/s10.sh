timeout -s KILL 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "config3" > gpurun_out/s10.log 2>&1; echo rc=$?
tail -3 gpurun_out/s10.log
timeout -s KILL 900 python bench.py > gpurun_out/s10_bench.json 2> gpurun_out/s10_bench.err; echo bench=$?
head -c 3000 gpurun_out/s10_bench.json
