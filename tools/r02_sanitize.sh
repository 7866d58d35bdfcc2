# compute-sanitizer on the small workload (racecheck / synccheck / memcheck)
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_c1.py \
      > gpurun_out/r02_sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/r02_sanitize_$tool.log
done
TLRB_QRCP_BLOCKED=1 timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_c1.py \
    > gpurun_out/r02_sanitize_racecheck_blocked.log 2>&1
echo "racecheck blocked rc=$?"; tail -3 gpurun_out/r02_sanitize_racecheck_blocked.log
