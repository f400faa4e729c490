for n in a b c d e a; do echo "== $n"; for a in "4 1 3" "4 8 3"; do HZ_LIB=_v/lib$n.so timeout 300 python tools/prof_tm.py $a 2>&1 | tail -1; done; done
