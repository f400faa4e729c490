for n in b1 b05; do echo "== $n"; for k in 2 3 4c5; do HZ_LIB=_v/libm$n.so timeout -s KILL 300 python tools/precond_cmp.py $k 1 2>&1 | grep "precond=1"; done; done
