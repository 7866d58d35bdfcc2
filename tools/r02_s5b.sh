# session-5 call B: GEMM 16-byte copies A/B, K1 vector stores parity, C5 projection
mkdir -p gpurun_out
./tools/bench_gemm > gpurun_out/r02_gemm_bench_vec.txt 2>&1
TLRB_GEMM_NOVEC=1 ./tools/bench_gemm > gpurun_out/r02_gemm_bench_novec.txt 2>&1
paste -d'\n' gpurun_out/r02_gemm_bench_vec.txt gpurun_out/r02_gemm_bench_novec.txt
timeout 900 python -m pytest tests -x -q -m gpu -k "tile or matern or loglik or great or edge or dense" 2>&1 | tail -5 || exit 1
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-kriging > gpurun_out/r02_iter_bench.json 2> gpurun_out/r02_iter_bench.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r02_iter_bench.json").read().strip().splitlines()[-1])
print("value", d["value"], "e2e", d["e2e"]["value"], "parity", d["parity"]["rel"], "dom", d["roofline"]["kernel"],
      d["roofline"]["frac"], "step_roof", d["step_roofline"]["frac"])
for k, v in d.get("variants", {}).items(): print(k, v["s"], v["rel"])
for k, v in d["kernels"].items(): print(k, round(v["busy_ms_per_step"]), round(v["ms_per_step"]), v["launches_per_step"])
PY
timeout 2700 python tools/project_c5.py --lead 24 48 72 > gpurun_out/r02_c5.json 2> gpurun_out/r02_c5.log
tail -c 1500 gpurun_out/r02_c5.json; tail -5 gpurun_out/r02_c5.log
