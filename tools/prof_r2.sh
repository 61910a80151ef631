#!/bin/bash
# Round-2 ncu evidence: launch list of a quick bench run + full captures of the
# scheduled engine's three kernels (plan, salvage copy, merge) at 2^30 int32.
set -x
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 1 --quick > gpurun_out/r2_quick.json 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches.csv \
    python bench.py --steps 2 --warmup 1 --quick > gpurun_out/r2_ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"^k_flow$|k_flow_save|k_flow_plan" -s 3 -c 3 \
    -o gpurun_out/r2_flow_full python tools/prof_flow.py 29 auto 3 > gpurun_out/r2_flow_full.log 2>&1
