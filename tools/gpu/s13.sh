timeout -s KILL 900 python -m pytest tests/test_gpu_cbs.py -v -s -p no:cacheprovider -k table2 > gpurun_out/s13.log 2>&1; echo rc=$?
grep -E "PASS|FAIL|Error|CBS|err vs|G4|passed|failed|assert" gpurun_out/s13.log | head -30
