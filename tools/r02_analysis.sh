# DGEMM ncu (ours vs cuBLAS on the 4096^3 and batched 760^3 shapes) and the C3 TLR timeline / per-step trace
mkdir -p gpurun_out
BENCH_SHAPE=9 ./tools/bench_gemm > gpurun_out/r02a_gemm9.txt 2>&1 || exit 1
for sh in 9 7 5; do
  BENCH_SHAPE=$sh timeout 600 ncu --set full --clock-control none --import-source on -c 4 \
     -o gpurun_out/r02a_gemm_shape$sh ./tools/bench_gemm > gpurun_out/r02a_ncu_gemm$sh.log 2>&1
  echo "ncu shape $sh rc=$?"
done
timeout 900 python tools/timeline_cfg.py C3 --bucket 100 > gpurun_out/r02a_timeline_c3.txt 2>&1
echo "timeline rc=$?"; head -20 gpurun_out/r02a_timeline_c3.txt
TLRB_TRACE=1 timeout 900 python tools/trace_cfg.py C3 > gpurun_out/r02a_trace_c3.out 2> gpurun_out/r02a_trace_c3.log
echo "trace rc=$?"; tail -3 gpurun_out/r02a_trace_c3.out
