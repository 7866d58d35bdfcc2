#!/bin/bash
# ncu recipe (B200_PROFILING.md): plain run first, then the launch list, then
# one --set full capture of the dominant kernels.  Run under gpurun.
set -e
CMD="python bench.py --steps 1 --warmup 1 --no-variants --no-cpu"
mkdir -p gpurun_out
$CMD > gpurun_out/plain.json 2> gpurun_out/plain.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"jacobi|qrcp|dgemm" \
    -s 40 -c 6 -o gpurun_out/prof_full $CMD > gpurun_out/ncu_full.log 2>&1
