for sh in 2 5; do for c in 3 4 5 7 8; do echo "shape $sh cfg $c: $(BENCH_SHAPE=$sh TLRB_GEMM_CFG=$c ./tools/bench_gemm | cut -c1-75)"; done; done
./tools/bench_gemm | cut -c1-120
bash tools/r02_s5i.sh
