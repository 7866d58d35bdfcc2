#!/bin/bash
set -e
CMD="python bench.py --steps 1 --warmup 1 --no-variants --no-cpu"
$CMD > gpurun_out/plain3.json 2> gpurun_out/plain3.err
ncu --set full --clock-control none --import-source on -k regex:jacobi_cluster -s 8 -c 1 \
    -o gpurun_out/prof_jacobi2 $CMD > gpurun_out/ncu_jacobi2.log 2>&1
