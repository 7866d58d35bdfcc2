# session-5 call E: factored path over the dense limit + split GEMM batches: bench iteration, A/B, tests
mkdir -p gpurun_out
run() {  # tag, env...
  tag=$1; shift
  env "$@" timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-kriging --no-variants > gpurun_out/r02_iter_$tag.json 2> gpurun_out/r02_iter_$tag.err
  python - "$tag" <<'PY'
import json, sys
tag = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/r02_iter_{tag}.json").read().strip().splitlines()[-1])
except Exception as e:
    print(tag, "FAILED", e); print(open(f"gpurun_out/r02_iter_{tag}.err").read()[-800:]); sys.exit(0)
print(tag, "value", round(d["value"], 4), "e2e", round(d["e2e"]["value"], 4), "parity", d["parity"]["rel"], "launches", d["gpu_launches"],
      "dense_tiles/max_rank", d["work"].get("max_rank"), "arena", d["work"]["arena_peak_gb"])
print("   ", {k: (round(v["busy_ms_per_step"]), v["launches_per_step"]) for k, v in d["kernels"].items()})
PY
}
run base A=1
run nosplit TLRB_GEMM_SPLIT=0
run noover TLRB_FACTORED_OVER=0
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -8
timeout 2400 python tools/project_c5.py --lead 24 48 72 > gpurun_out/r02_c5.json 2> gpurun_out/r02_c5.log
tail -c 1800 gpurun_out/r02_c5.json; tail -3 gpurun_out/r02_c5.log | cut -c1-300
