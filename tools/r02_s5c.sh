# session-5 call C: iteration bench (batched zero fill, work model), GEMM shape stats at C3, ncu of the GEMM tile configs
mkdir -p gpurun_out
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-kriging > gpurun_out/r02_iter_bench.json 2> gpurun_out/r02_iter_bench.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r02_iter_bench.json").read().strip().splitlines()[-1])
print("value", d["value"], "e2e", d["e2e"]["value"], "parity", d["parity"]["rel"], "dom", d["roofline"]["kernel"],
      d["roofline"]["frac"], "step_roof", d["step_roofline"]["frac"], "launches", d["gpu_launches"])
for k, v in d.get("variants", {}).items(): print(k, v["s"], v["rel"])
for k, v in d["kernels"].items(): print(k, round(v["busy_ms_per_step"]), round(v["ms_per_step"]), v["launches_per_step"])
print(d["profiled_step"])
PY
TLRB_GEMM_STATS=1 timeout 600 python tools/trace_cfg.py C3 --no-warm > gpurun_out/r02_gemm_stats_c3.txt 2>&1
grep gemm-stats gpurun_out/r02_gemm_stats_c3.txt | sort -k9 -n -r | head -40
TLRB_TRACE=1 timeout 600 python tools/trace_cfg.py C3 > gpurun_out/r02_trace_c3.txt 2>&1
python tools/trace_sum.py gpurun_out/r02_trace_c3.txt 2>&1 | tail -30
for spec in "dgemm_tiles_kernel<64, 64:200:2" "dgemm_tiles_kernel<64, 128:200:2" "dgemm_tiles_kernel<128:20:2"; do
  IFS=: read -r re skip cnt <<< "$spec"
  tag=$(echo "$re" | tr -d '<, ' )
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$re" -s $skip -c $cnt \
      -o gpurun_out/r02_full_$tag python tools/trace_cfg.py C3 --no-warm > gpurun_out/r02_ncu_full_$tag.log 2>&1
  echo "$tag rc=$?"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dgemm_tiles_kernel<128" -s 60 -c 2 \
      -o gpurun_out/r02_full_dense_gemm128 python tools/trace_cfg.py C3 --no-warm --dense > gpurun_out/r02_ncu_full_dense128.log 2>&1
echo "dense128 rc=$?"
