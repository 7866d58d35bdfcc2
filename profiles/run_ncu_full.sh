#!/bin/bash
# --set full captures of the two dominant kernels (after a clean plain run).
set -e
CMD="python bench.py --steps 1 --warmup 1 --no-variants --no-cpu"
mkdir -p gpurun_out
$CMD > gpurun_out/plain2.json 2> gpurun_out/plain2.err
ncu --set full --clock-control none --import-source on -k regex:jacobi_cluster -s 6 -c 2 \
    -o gpurun_out/prof_jacobi $CMD > gpurun_out/ncu_jacobi.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:qrcp -s 2 -c 1 \
    -o gpurun_out/prof_qrcp $CMD > gpurun_out/ncu_qrcp.log 2>&1
