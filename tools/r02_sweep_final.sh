# session-5 call O: storage-threshold sweep with the final kernels; DMMA pipe of the final GEMM (microbench shapes)
mkdir -p gpurun_out
out=gpurun_out/r02_sweep_final.jsonl; : > $out
for r in 0.3 0.25 0.2 0.15 0.1; do
  TLRB_DENSE_FRAC=$r timeout 300 python tools/c3_once.py >> $out 2>> gpurun_out/r02_sweep_final.err
done
cat $out | cut -c1-330
for sh in 9 7 0; do
  BENCH_SHAPE=$sh timeout 600 ncu --set full --clock-control none -k regex:dgemm_tiles -s 2 -c 1 \
     -o gpurun_out/r02_full_gemmbench_shape$sh ./tools/bench_gemm > gpurun_out/r02_ncu_gemmbench$sh.log 2>&1
  echo "shape $sh rc=$?"
done
python tools/ncu_rep_table.py gpurun_out/r02_full_gemmbench_shape*.ncu-rep > gpurun_out/r02_counters_gemmbench.md 2>&1
cat gpurun_out/r02_counters_gemmbench.md | cut -c1-260
