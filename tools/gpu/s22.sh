# r-hat through TMA in the dot epilogues: solve-iteration A/B on config 4, then the solve/parity suites
for L in _v/libbase.so _v/librh.so _v/libbase.so _v/librh.so; do
  echo "== $L"; HZ_LIB=$L timeout -s KILL 300 python tools/prof_solve.py 20 1 2 | tail -1
done > gpurun_out/s22_ab.log 2>&1
for L in _v/libbase.so _v/librh.so; do
  echo "== $L ell2"; HZ_LIB=$L timeout -s KILL 300 python tools/prof_solve.py 20 2 2 | tail -1
done >> gpurun_out/s22_ab.log 2>&1
cat gpurun_out/s22_ab.log
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -8 > gpurun_out/s22_pytest.log
cat gpurun_out/s22_pytest.log
