# halo-overlapped apply: loopback + parity suites; A/B of the accumulation tree on config 4
timeout -s KILL 900 python -m pytest tests/test_gpu_loopback.py tests/test_gpu_parity.py -x -q 2>&1 | tail -8 > gpurun_out/s19_pytest.log
for n in 1 8; do
  for L in paper_2108_08730_b200/libhz.so _v/libtree.so; do
    echo "== $L"; HZ_LIB=$L timeout -s KILL 300 python tools/prof_tm.py 4 $n 3
  done
done > gpurun_out/s19_ab.log 2>&1
for n in 1 8; do
  for L in _v/libtree.so paper_2108_08730_b200/libhz.so; do
    echo "== $L"; HZ_LIB=$L timeout -s KILL 300 python tools/prof_tm.py 4 $n 3
  done
done >> gpurun_out/s19_ab.log 2>&1
cat gpurun_out/s19_pytest.log gpurun_out/s19_ab.log
