# round-2 re-entry verification: GEMM microbench, GPU tests, sanitizers, bench
mkdir -p gpurun_out
./tools/bench_gemm > gpurun_out/r02_gemm_bench.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -30 > gpurun_out/r02_gputests.log
tail -5 gpurun_out/r02_gputests.log
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_c1.py \
      > gpurun_out/r02_sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/r02_sanitize_$tool.log
done
TLRB_QRCP_BLOCKED=1 timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_c1.py \
    > gpurun_out/r02_sanitize_racecheck_blocked.log 2>&1
echo "racecheck blocked rc=$?"; tail -3 gpurun_out/r02_sanitize_racecheck_blocked.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r02_bench_c3.json 2> gpurun_out/r02_bench_c3.err
tail -c 1500 gpurun_out/r02_bench_c3.json; tail -3 gpurun_out/r02_bench_c3.err
