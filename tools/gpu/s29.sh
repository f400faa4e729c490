# early producer start + float4 table staging: A/B against the previous kernel on small and large grids, then the GPU suite
for L in _variants/base/libhz.so paper_2108_08730_b200/libhz.so _variants/base/libhz.so paper_2108_08730_b200/libhz.so; do
  echo "== $L"
  for c in 1 2 3 4; do HZ_LIB=$L timeout -s KILL 200 python tools/prof_tm.py $c 1 3 | tail -1; done
  HZ_LIB=$L timeout -s KILL 200 python tools/prof_tm.py 2 4 3 | tail -1
  HZ_LIB=$L timeout -s KILL 200 python tools/prof_tm.py 4 8 3 | tail -1
done > gpurun_out/s29_ab.log 2>&1
cat gpurun_out/s29_ab.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s29_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/s29_tests.log
timeout 1200 python bench.py > gpurun_out/s29_bench.json 2> gpurun_out/s29_bench.err; echo bench=$?
