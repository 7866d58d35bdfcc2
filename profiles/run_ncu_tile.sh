#!/bin/bash
set -e
python tools/one_tile.py > gpurun_out/one_tile.txt 2>&1
TLRB_JACOBI_MAXCL=1 python tools/one_tile.py > gpurun_out/one_tile_cl1.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:"jacobi|qrcp" -s 2 -c 2 \
    -o gpurun_out/prof_tile python tools/one_tile.py > gpurun_out/ncu_tile.log 2>&1
