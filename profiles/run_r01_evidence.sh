#!/bin/bash
# Round-1 evidence: GPU tests, bench line (+ reference arm), launch list of
# the bench command, DRAM traffic of every Jacobi launch of the timed step
# (metrics-only pass, CSV) and --set full of two of them.  Outputs stay
# small (gpurun copies back <= 64 MiB).
set -e
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/ev_pytest.log 2>&1 || true
python bench.py > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err
python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/ev_bench_ref.json 2> gpurun_out/ev_bench_ref.err
CMD="python bench.py --steps 1 --warmup 3 --no-variants --no-cpu"
$CMD > gpurun_out/ev_plain.json 2> gpurun_out/ev_plain.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/ev_launches.csv $CMD > gpurun_out/ev_ncu_launches.log 2>&1
# the timed step's Jacobi launches: 3 warm-up evaluations x 68 precede it
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
    -k regex:jacobi_cluster -s 204 -c 68 --log-file gpurun_out/ev_jacobi_dram.csv $CMD > gpurun_out/ev_ncu_dram.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:jacobi_cluster -s 204 -c 2 \
    -o gpurun_out/ev_jacobi_full $CMD > gpurun_out/ev_ncu_full.log 2>&1
ncu -i gpurun_out/ev_jacobi_full.ncu-rep --page raw --csv > gpurun_out/ev_jacobi_full_raw.csv 2>/dev/null || true
tail -n2 gpurun_out/ev_pytest.log
du -sh gpurun_out
