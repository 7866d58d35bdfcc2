# one build -> measure iteration on the GPU box: bench line (no CPU baseline) + the GPU test suite
mkdir -p gpurun_out
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu --no-kriging > gpurun_out/r02_iter_bench.json 2> gpurun_out/r02_iter_bench.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r02_iter_bench.json").read().strip().splitlines()[-1])
print("value", d["value"], "e2e", d["e2e"]["value"], "parity", d["parity"]["rel"], "dom", d["roofline"]["kernel"],
      d["roofline"]["frac"], "step_roof", d["step_roofline"]["frac"], "launches", d["gpu_launches"], d["phases_ms"])
for k, v in d.get("variants", {}).items(): print(k, v["s"], v["rel"])
print({k: (round(v["busy_ms_per_step"]), v["launches_per_step"]) for k, v in d["kernels"].items()})
PY
timeout 1800 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
