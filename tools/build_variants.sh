#!/bin/bash
# Build A/B variants of libwsb200.so in parallel: tools/build_variants.sh name1="-DX -DY" name2="..."  -> build/lib_<name>.so
# Load one with WSB_LIB=build/lib_<name>.so (tools/perf_probe.py, bench.py).
cd "$(dirname "$0")/.." || exit 1
mkdir -p build
for spec in "$@"; do
  name="${spec%%=*}"; flags="${spec#*=}"
  ( WSB_NVCC_EXTRA="$flags" python -m paper_2205_07610_b200.build -o "$PWD/build/lib_$name.so" > build/lib_$name.log 2>&1 && echo "built $name" || echo "FAILED $name" ) &
done
wait
