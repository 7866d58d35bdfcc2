# C3 GEMM shape statistics (TLR and dense) + per-class profile of a dense evaluation (diagnostic runs)
TLRB_GEMM_STATS=1 timeout 600 python tools/trace_cfg.py C3 --no-warm > gpurun_out/r02_c3_gemm.out 2> gpurun_out/r02_c3_gemm.log
TLRB_GEMM_STATS=1 timeout 600 python tools/trace_cfg.py C3 --no-warm --dense > gpurun_out/r02_c3_gemm_dense.out 2> gpurun_out/r02_c3_gemm_dense.log
timeout 600 python tools/trace_cfg.py C3 --dense --profile > gpurun_out/r02_c3_dense_prof.out 2>&1
timeout 600 python tools/trace_cfg.py C3 --profile > gpurun_out/r02_c3_tlr_prof.out 2>&1
cat gpurun_out/r02_c3_dense_prof.out gpurun_out/r02_c3_tlr_prof.out
for f in gpurun_out/r02_c3_gemm.log gpurun_out/r02_c3_gemm_dense.log; do echo $f; grep gemm-stats $f | sort -k8 -g -r | head -16; done
