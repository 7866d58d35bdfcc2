mkdir -p gpurun_out
./tools/bench_gemm > gpurun_out/r02_gemm_bench_vec.txt 2>&1
TLRB_GEMM_NOVEC=1 ./tools/bench_gemm > gpurun_out/r02_gemm_bench_novec.txt 2>&1
paste -d'\n' gpurun_out/r02_gemm_bench_vec.txt gpurun_out/r02_gemm_bench_novec.txt
