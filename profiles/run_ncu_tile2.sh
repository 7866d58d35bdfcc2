#!/bin/bash
# one C2 offset-1 tile: source-level capture of the QRCP-cluster and Jacobi kernels
set -e
python tools/one_tile.py > gpurun_out/one_tile.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:"jacobi|qrcp" -s 2 -c 2 \
    -o gpurun_out/prof_tile2 python tools/one_tile.py > gpurun_out/ncu_tile2.log 2>&1
