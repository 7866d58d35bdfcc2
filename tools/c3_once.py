"""One C3 configuration (bench workload: z_c3 fixture, TLR 1e-7, cap 380):
two evaluations, prints the best time, ll, relative gap to the reference
dense ll and the storage statistics as one JSON line.  Knobs come from the
environment (TLRB_*), e.g. a sweep:
    for r in 0.45 0.3; do TLRB_DENSE_FRAC=$r python tools/c3_once.py; done"""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1804_09137_b200 as tb  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
n, nb, cap, acc, theta = (62_500, 760, 380, 1e-7, (1.0, 0.03, 0.5)) if cfg == "C3" else \
    (10_000, 500, 0, 1e-9, (1.0, 0.1, 0.5))
z = np.load(ROOT / "tests/golden" / ("z_c3.npz" if cfg == "C3" else "z_big.npz"))[cfg]
ref = (json.loads((ROOT / "tests/golden/c3.json").read_text())["C3"]["modes"]["dense"]["ll"] if cfg == "C3"
       else -2792.8552965835443)
h = tb.Handle(tb.generate_locations(n, 0).coords, nb, max_rank=cap)
p = tb.MaternParams(*theta)
ts, ll = [], None
for _ in range(int(os.environ.get("REPS", "2"))):
    t0 = time.perf_counter()
    ll = h.loglik(z, p, acc)[0]
    ts.append(time.perf_counter() - t0)
st = h.last_stats
rm = h.rank_map()
low = np.tril(rm, -1)
print(json.dumps({"cfg": cfg, "env": {k: v for k, v in os.environ.items() if k.startswith("TLRB_")},
                  "s": min(ts), "ll": ll, "rel_vs_ref": abs(ll - ref) / abs(ref),
                  "dense_tiles": int((low == -1).sum()), "max_rank": st["max_rank"],
                  "arena_gb": st["arena_peak_bytes"] / 1e9, "launches": st["kernel_launches"],
                  "phases": {k: round(st[k]) for k in ("ms_generate", "ms_compress", "ms_factor", "ms_solve")}}),
      flush=True)
