#!/bin/bash
# One GPU call that refreshes the per-round evidence under gpurun_out/ (copied to profiles/ by hand afterwards).
R=${1:-r02}
for w in cfg2 cfg1 cfg3 cfg4 cfg5; do
  python bench.py --workload $w --steps 10 --warmup 3 2>/dev/null | tail -1 > gpurun_out/${R}_bench_$w.json
  cut -c1-160 gpurun_out/${R}_bench_$w.json
done
python bench.py --workload cfg1 --pairs 1000000 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/${R}_bench_cfg1_1M.json
python bench.py --impl reference --steps 3 --warmup 1 2>/dev/null | tail -1 > gpurun_out/${R}_bench_reference_arm_cfg2.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${R}_launches_bench_cfg2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${R}_launches_cfg3.csv python bench.py --workload cfg3 --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:s16_local -s 1 -c 1 -f -o gpurun_out/${R}_ncu_s16_local python tools/perf_probe.py --variants s16x2 --reps 2 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:s16_global -s 1 -c 1 -f -o gpurun_out/${R}_ncu_s16_global python tools/perf_probe.py --type global --gap linear --variants auto --reps 2 > /dev/null 2>&1
ls -la gpurun_out | tail -12
