# register-cap / ptxas variants of the shipped apply27_tm (12 warps): does another schedule of the same code run faster?
for V in base n160 n152 n144 n136 po2 base; do
  L=_variants/$V/libhz.so
  echo "== $V"
  HZ_LIB=$L timeout -s KILL 200 python tools/prof_tm.py 4 1 3 | tail -1
  HZ_LIB=$L timeout -s KILL 200 python tools/prof_tm.py 4 8 3 | tail -1
  HZ_LIB=$L timeout -s KILL 200 python tools/prof_tm.py 4 1 3 0 | tail -1
done > gpurun_out/s30_sweep.log 2>&1
cat gpurun_out/s30_sweep.log
