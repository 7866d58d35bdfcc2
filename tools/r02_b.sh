mkdir -p gpurun_out
for c in 0 1 2; do echo "cfg $c"; TLRB_GEMM_CFG=$c ./tools/bench_gemm; done > gpurun_out/r02b_gemm_cfgs.txt 2>&1
cat gpurun_out/r02b_gemm_cfgs.txt
timeout 900 python tools/timeline_cfg.py C3 --bucket 100 > gpurun_out/r02b_timeline_c3.txt 2>&1
echo "timeline rc=$?"; head -40 gpurun_out/r02b_timeline_c3.txt
TL_WINDOW="2000,2200" timeout 900 python tools/timeline_cfg.py C3 --bucket 1000 > gpurun_out/r02b_timeline_c3_win.txt 2>&1
echo "win rc=$?"
