# C3 step trace + GEMM shape statistics (diagnostic runs, serialising)
TLRB_TRACE=1 timeout 600 python tools/trace_cfg.py C3 > gpurun_out/r02_c3_trace.out 2> gpurun_out/r02_c3_trace.log
TLRB_GEMM_STATS=1 timeout 600 python tools/trace_cfg.py C3 --no-warm > gpurun_out/r02_c3_gemm.out 2> gpurun_out/r02_c3_gemm.log
grep -c step gpurun_out/r02_c3_trace.log; tail -3 gpurun_out/r02_c3_trace.out; grep gemm-stats gpurun_out/r02_c3_gemm.log | sort -k7 -n -r | head -30
