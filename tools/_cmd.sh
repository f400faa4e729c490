timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
for c in "5 1 c64" "5 1 c64 20 0" "2 4 c64"; do python tools/prof_apply.py $c | cut -c1-150; done
for c in "5 1 c64" "5 1 c64 20 0" "2 4 c64"; do HZ_LIB=$PWD/_variants/m3/libhz.so python tools/prof_apply.py $c | cut -c1-150; done
HZ_LIB=$PWD/_variants/m3/libhz.so python tools/prof_apply.py 5 1 c64 3 0 > gpurun_out/plain.log 2>&1 && HZ_LIB=$PWD/_variants/m3/libhz.so ncu --set full --clock-control none --import-source on -k regex:apply27 -s 6 -c 2 -o gpurun_out/prof_m3 python tools/prof_apply.py 5 1 c64 3 0 > gpurun_out/ncu5.log 2>&1; tail -1 gpurun_out/ncu5.log
