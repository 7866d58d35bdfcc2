# one build -> measure iteration on the GPU box
./tools/bench_gemm > gpurun_out/r02_gemm_bench.txt 2>&1
cat gpurun_out/r02_gemm_bench.txt
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -15 > gpurun_out/r02_iter_tests.log
tail -5 gpurun_out/r02_iter_tests.log
timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu --no-kriging > gpurun_out/r02_iter_bench.json 2> gpurun_out/r02_iter_bench.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r02_iter_bench.json").read().strip().splitlines()[-1])
print("value", d["value"], "e2e", d["e2e"]["value"], "parity", d["parity"]["rel"], "dom", d["roofline"]["kernel"],
      d["roofline"]["frac"], "step_roof", d["step_roofline"]["frac"])
for k, v in d.get("variants", {}).items(): print(k, v["s"], v["rel"])
for k, v in d["kernels"].items(): print(k, round(v["busy_ms_per_step"]), round(v["ms_per_step"]), v["launches_per_step"])
PY
