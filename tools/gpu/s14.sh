timeout 200 python tools/cbs_vs_fd.py 3 model 5 -1 1.0 3.5 2>&1 | tail -1
timeout 200 python tools/cbs_vs_fd.py 3 model 5 -1 1.0 7.0 50 2>&1 | tail -1
timeout 200 python tools/cbs_vs_fd.py 3 model 5 -1 1.0 14.0 2>&1 | tail -1
