#!/bin/bash
# Build apply-kernel tuning variants into _variants/<name>/libhz.so (HZ_LIB selects one at run time).
cd "$(dirname "$0")/.."
build() {
  name=$1; shift
  mkdir -p _variants/$name
  HZ_BUILD_DIR=_variants/$name/obj HZ_LIB=$PWD/_variants/$name/libhz.so HZ_EXTRA_NVCC="$*" python -c "
import importlib.util
spec=importlib.util.spec_from_file_location('b','paper_2108_08730_b200/build.py'); b=importlib.util.module_from_spec(spec); spec.loader.exec_module(b); b.build(force=True)" || echo "FAILED $name"
}
for v in "$@"; do
  IFS=: read name flags <<< "$v"
  build $name $flags &
done
wait
