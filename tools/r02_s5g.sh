# session-5 call G: blocked TRSM on DMMA + dense look-ahead: bench with variants, new tests, GEMM ncu
mkdir -p gpurun_out
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu --no-kriging > gpurun_out/r02_iter_bench.json 2> gpurun_out/r02_iter_bench.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r02_iter_bench.json").read().strip().splitlines()[-1])
print("value", d["value"], "e2e", d["e2e"]["value"], "parity", d["parity"]["rel"], "dom", d["roofline"]["kernel"],
      d["roofline"]["frac"], "step_roof", d["step_roofline"]["frac"], "launches", d["gpu_launches"])
for k, v in d.get("variants", {}).items(): print(k, v["s"], v["rel"])
print({k: (round(v["busy_ms_per_step"]), v["launches_per_step"]) for k, v in d["kernels"].items()})
PY
TLRB_TRSM_BLOCKED=0 TLRB_LOOKAHEAD=0 timeout 300 python tools/trace_cfg.py C3 --dense 2>&1 | grep "^ll" | cut -c1-120
timeout 300 python tools/trace_cfg.py C3 --dense 2>&1 | grep "^ll" | cut -c1-120
TLRB_TRSM_BLOCKED=64 timeout 300 python tools/trace_cfg.py C3 --dense 2>&1 | grep "^ll" | cut -c1-120
timeout 1500 python -m pytest tests -x -q -m gpu -k "c3_full or arena or lookahead or dense or solves or multigpu or max_rank" 2>&1 | tail -8
bash tools/r02_s5f.sh
