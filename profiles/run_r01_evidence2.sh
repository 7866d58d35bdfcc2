#!/bin/bash
# Final round-1 evidence with the final code: GPU tests, smoke, bench line,
# reference arm, launch list of the bench command, Jacobi DRAM traffic of the
# timed step, --set full of two Jacobi launches (outputs stay small).
set -e
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/e2_pytest.log 2>&1 || true
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e2_smoke.log 2>&1 || true
python bench.py > gpurun_out/e2_bench.json 2> gpurun_out/e2_bench.err
python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/e2_bench_ref.json 2> gpurun_out/e2_bench_ref.err
CMD="python bench.py --steps 1 --warmup 3 --no-variants --no-cpu"
$CMD > gpurun_out/e2_plain.json 2> gpurun_out/e2_plain.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/e2_launches.csv $CMD > gpurun_out/e2_ncu_launches.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
    -k regex:jacobi_cluster -s 204 -c 68 --log-file gpurun_out/e2_jacobi_dram.csv $CMD > gpurun_out/e2_ncu_dram.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:jacobi_cluster -s 204 -c 2 \
    -o gpurun_out/e2_jacobi_full $CMD > gpurun_out/e2_ncu_full.log 2>&1
tail -n2 gpurun_out/e2_pytest.log; cat gpurun_out/e2_smoke.log
du -sh gpurun_out
