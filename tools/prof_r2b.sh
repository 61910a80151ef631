#!/bin/bash
# Round-2 (late) evidence: full bench line, reference arm, config 3/4 legs, the
# launch list of a quick run, and ncu --set full of the scheduled engine's kernels.
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err || exit 1
python bench.py --impl reference > gpurun_out/r2b_reference.json 2> gpurun_out/r2b_reference.err
python bench.py --cfg 3 > gpurun_out/r2b_cfg3.json 2> gpurun_out/r2b_cfg3.err
python bench.py --cfg 4 > gpurun_out/r2b_cfg4.json 2> gpurun_out/r2b_cfg4.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2b_launches.csv \
    python bench.py --steps 2 --warmup 1 --quick > gpurun_out/r2b_ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"^k_flow$|k_flow_save|k_flow_plan" -s 3 -c 3 \
    -o gpurun_out/r2b_flow_full python tools/prof_flow.py 29 auto 3 > gpurun_out/r2b_flow_full.log 2>&1
