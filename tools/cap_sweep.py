"""C2 log-likelihood time / parity vs the storage cap (max_rank):
    python tools/cap_sweep.py 1e-9 0 250 200 150"""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import json  # noqa: E402
import paper_1804_09137_b200 as tb  # noqa: E402

acc = float(sys.argv[1])
caps = [int(c) for c in sys.argv[2:]]
ref = json.loads((ROOT / "tests/golden/loglik_big.json").read_text())
locs = tb.generate_locations(10000, 0)
z = np.load(ROOT / "tests/golden/z_big.npz")["C2"]
p = tb.MaternParams(1.0, 0.1, 0.5)
gold = None
for key in ("loglik",):
    pass
for cap in caps:
    h = tb.Handle(locs.coords, 500, max_rank=cap)
    h.loglik(z, p, acc)
    ts = []
    for _ in range(2):
        t0 = time.perf_counter()
        ll = h.loglik(z, p, acc)[0]
        ts.append(time.perf_counter() - t0)
    rm = h.rank_map()
    print(f"acc {acc:g} cap {cap}: ll {ll!r} wall {min(ts):.3f} s dense tiles {(rm < 0).sum()} "
          f"max_rank {h.last_stats['max_rank']} stored {h.last_stats['stored_reals']/1e6:.1f}M", flush=True)
    h.close()
