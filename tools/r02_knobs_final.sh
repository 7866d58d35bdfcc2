mkdir -p gpurun_out
out=gpurun_out/r02_knobs_final.jsonl; : > $out
python tools/c3_once.py >> $out 2>/dev/null
TLRB_TRSM_BLOCKED=64 python tools/c3_once.py >> $out 2>/dev/null
TLRB_TRSM_BLOCKED=256 python tools/c3_once.py >> $out 2>/dev/null
TLRB_FACTORED_ORTHO=0 python tools/c3_once.py >> $out 2>/dev/null
TLRB_GEMM_SPLIT=0 python tools/c3_once.py >> $out 2>/dev/null
TLRB_LOOKAHEAD=0 python tools/c3_once.py >> $out 2>/dev/null
python - <<'PY'
import json
for l in open("gpurun_out/r02_knobs_final.jsonl"):
    d = json.loads(l); print(d["env"], round(d["s"], 4), d["rel_vs_ref"], d["launches"], d["phases"])
PY
