# no-producer apply27_tm (12 consumer warps, last releaser refills): A/B vs the committed build, then parity
for n in 1 8; do
  for L in _v/libbase.so _v/libnoprod.so _v/libbase.so _v/libnoprod.so; do
    echo "== $L"; HZ_LIB=$L timeout -s KILL 300 python tools/prof_tm.py 4 $n 3
  done
done > gpurun_out/s20_ab.log 2>&1
cat gpurun_out/s20_ab.log
timeout -s KILL 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py tests/test_gpu_solve.py -x -q 2>&1 | tail -8 > gpurun_out/s20_pytest.log
cat gpurun_out/s20_pytest.log
