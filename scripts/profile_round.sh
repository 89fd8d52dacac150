#!/bin/bash
# Round profile on one B200 (run under gpurun from the repo root; writes gpurun_out/):
#   1. bench lines of the five configs (default bench command, oracle cpu_baseline)
#   2. the launch list of config 4 (host-loop hook: ncu cannot see kernel nodes of
#      conditional graphs), gpu__time_duration per launch, clocks not locked
#   3. one `ncu --set full` capture of the persistent pass of configs 4 and 3
# Numbers printed under ncu are never bench values.
set -u
R=${1:-r02}
mkdir -p gpurun_out
for c in 4 3 5 1 2; do
  timeout 400 python bench.py --config $c > gpurun_out/${R}_bench_config$c.json 2> gpurun_out/${R}_bench_config$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${R}_c4_launches.csv \
  python bench.py --config 4 --hostloop --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${R}_c4_ncu_launches.log 2>&1
# first persistent pass launch of a config-4 call (passes 1-11 of the first attempt)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_inner_3d -c 1 \
  -o gpurun_out/${R}_c4_inner -f python scripts/profile_run.py --config 4 > gpurun_out/${R}_c4_ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_inner_2d -s 2 -c 1 \
  -o gpurun_out/${R}_c3_inner -f python scripts/profile_run.py --config 3 > gpurun_out/${R}_c3_ncu_full.log 2>&1
# summaries on the box (the two reports together exceed what gpurun brings back); KEEP_REPS=1 keeps them
python scripts/ncu_summary.py gpurun_out/${R}_c4_inner.ncu-rep 20 > gpurun_out/${R}_c4_inner_summary.txt 2>&1
python scripts/ncu_summary.py gpurun_out/${R}_c3_inner.ncu-rep 20 > gpurun_out/${R}_c3_inner_summary.txt 2>&1
[ "${KEEP_REPS:-0}" = "1" ] || rm -f gpurun_out/${R}_c4_inner.ncu-rep gpurun_out/${R}_c3_inner.ncu-rep
echo done
