#!/bin/bash
# Build A/B variants of libwsb200.so in parallel: tools/build_variants.sh name1="-DX -DY" name2="..."  -> build/lib_<name>.so
# Load one with WSB_LIB=build/lib_<name>.so (tools/perf_probe.py, bench.py).
cd "$(dirname "$0")/.." || exit 1
mkdir -p build
for spec in "$@"; do
  name="${spec%%=*}"; flags="${spec#*=}"
  ( /usr/local/cuda/bin/nvcc $flags -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
      -o build/lib_$name.so paper_2205_07610_b200/csrc/wsb200.cu 2> build/lib_$name.log && echo "built $name" || echo "FAILED $name" ) &
done
wait
