mkdir -p gpurun_out
run() {
  tag=$1; shift
  env "$@" timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-kriging --no-variants > gpurun_out/r02_iter_$tag.json 2> gpurun_out/r02_iter_$tag.err
  python - "$tag" <<'PY'
import json, sys
tag = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/r02_iter_{tag}.json").read().strip().splitlines()[-1])
except Exception as e:
    print(tag, "FAILED", e); print(open(f"gpurun_out/r02_iter_{tag}.err").read()[-1500:]); sys.exit(0)
print(tag, "value", round(d["value"], 4), "e2e", round(d["e2e"]["value"], 4), "parity", d["parity"]["rel"], "launches", d["gpu_launches"],
      "max_rank", d["work"].get("max_rank"), "arena", d["work"]["arena_peak_gb"], "dom", d["roofline"]["kernel"], round(d["roofline"]["frac"], 4))
print("   ", {k: (round(v["busy_ms_per_step"]), v["launches_per_step"]) for k, v in d["kernels"].items()})
PY
}
run ortho A=1
run noortho TLRB_FACTORED_ORTHO=0
timeout 1800 python -m pytest tests -x -q -m gpu 2>&1 | tail -8
