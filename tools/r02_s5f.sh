# session-5 call F: ncu --set full of the 128x128 GEMM (4096^3 and the 82 x 760^3 batch), with source
mkdir -p gpurun_out
for sh in 9 7; do
  BENCH_SHAPE=$sh ./tools/bench_gemm > gpurun_out/r02f_gemm$sh.txt 2>&1 || exit 1
  cat gpurun_out/r02f_gemm$sh.txt
  BENCH_SHAPE=$sh timeout 600 ncu --set full --clock-control none --import-source on -k regex:dgemm_tiles -s 2 -c 1 \
     -o gpurun_out/r02f_gemm_shape$sh ./tools/bench_gemm > gpurun_out/r02f_ncu_gemm$sh.log 2>&1
  echo "shape $sh rc=$?"
done
