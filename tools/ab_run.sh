#!/bin/bash
# run the kernel-only probe against each build/lib_<name>.so given as arguments (on the GPU box); extra env via ENVV
for name in "$@"; do
  echo "== $name ${ENVV:-}"
  env ${ENVV:-} WSB_LIB=build/lib_$name.so python tools/perf_probe.py --variants ${PROBE_VARIANTS:-s16x2} --reps 4 ${PROBE_ARGS:-} 2>&1 | grep -v "^upload" | tail -3
done
