timeout -s KILL 300 python -m pytest tests/test_gpu_solve.py -v -x -p no:cacheprovider -k "not config3" > gpurun_out/s7.log 2>&1
echo rc=$?
