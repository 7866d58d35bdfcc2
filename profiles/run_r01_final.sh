#!/bin/bash
# Round-1 evidence: bench line (+ reference arm), launch list of the same
# command, --set full of the top kernels (Jacobi, blocked-QRCP panel/pick).
set -e
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
CMD="python bench.py --steps 1 --warmup 3 --no-variants --no-cpu"
$CMD > gpurun_out/plain_f.json 2> gpurun_out/plain_f.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_f.csv $CMD > gpurun_out/ncu_launches_f.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"jacobi_cluster|bq_panel|bq_pick" -s 6 -c 3 \
    -o gpurun_out/prof_f $CMD > gpurun_out/ncu_full_f.log 2>&1
