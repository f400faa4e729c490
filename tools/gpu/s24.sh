# apply27_tm tuning sweep: consumer warps (11 -> 15 at 128 registers), ring depth, q-sum FMA form
for V in base w15s8 w15s10 w15q w11q base w15s10; do
  L=_variants/$V/libhz.so
  echo "== $V"
  HZ_LIB=$L timeout -s KILL 200 python tools/prof_tm.py 4 1 3 | tail -1
  HZ_LIB=$L timeout -s KILL 200 python tools/prof_tm.py 4 8 3 | tail -1
  HZ_LIB=$L timeout -s KILL 200 python tools/prof_tm.py 4 1 3 0 | tail -1
  HZ_LIB=$L timeout -s KILL 300 python tools/prof_solve.py 20 1 2 | tail -1
done > gpurun_out/s24_sweep.log 2>&1
cat gpurun_out/s24_sweep.log
