#!/bin/bash
# --set full of the C3 Jacobi / QRCP launches in a throughput batch (after a plain run).
set -e
mkdir -p gpurun_out
CMD="python tools/trace_cfg.py C3 --no-warm"
$CMD > gpurun_out/c3_plain.out 2>&1
ncu --set full --clock-control none --import-source on -k regex:"jacobi_cluster" -s 12 -c 2 \
    -o gpurun_out/prof_c3_jacobi $CMD > gpurun_out/ncu_c3_jacobi.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"qrcp_kernel|bq_panel|bq_pick" -s 8 -c 4 \
    -o gpurun_out/prof_c3_qrcp $CMD > gpurun_out/ncu_c3_qrcp.log 2>&1
