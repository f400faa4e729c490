#!/bin/bash
# Run prof_apply for each built variant: tools/sweep.sh "CFG NRHS DT" ...
cd "$(dirname "$0")/.."
for d in _variants/*/; do
  n=$(basename $d)
  for c in "$@"; do
    echo -n "$n $c "; HZ_LIB=$PWD/$d/libhz.so python tools/prof_apply.py $c 2>&1 | tail -1
  done
done
