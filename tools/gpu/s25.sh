# apply27_tm: 2 rows per thread (2x2 points, 7 consumer warps at 255 registers) against the 1-row kernel
for V in base r2 r2q r2s12 base r2; do
  L=_variants/$V/libhz.so
  echo "== $V"
  HZ_LIB=$L timeout -s KILL 200 python tools/prof_tm.py 4 1 3 | tail -1
  HZ_LIB=$L timeout -s KILL 200 python tools/prof_tm.py 4 8 3 | tail -1
  HZ_LIB=$L timeout -s KILL 200 python tools/prof_tm.py 4 1 3 0 | tail -1
  HZ_LIB=$L timeout -s KILL 300 python tools/prof_solve.py 20 1 2 | tail -1 | cut -c1-60
done > gpurun_out/s25_sweep.log 2>&1
cat gpurun_out/s25_sweep.log
HZ_LIB=_variants/r2/libhz.so timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py -m gpu -x -q 2>&1 | tail -8 > gpurun_out/s25_pytest.log
cat gpurun_out/s25_pytest.log
