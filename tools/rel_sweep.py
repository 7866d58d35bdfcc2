"""Rank map / ll / time of one C2 TLR evaluation (compare TLRB_QRCP_REL settings):
    TLRB_QRCP_REL=0.1 python tools/rel_sweep.py 1e-9 out.npz"""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1804_09137_b200 as tb  # noqa: E402

acc = float(sys.argv[1])
locs = tb.generate_locations(10000, 0)
z = np.load(ROOT / "tests/golden/z_big.npz")["C2"]
h = tb.Handle(locs.coords, 500)
p = tb.MaternParams(1.0, 0.1, 0.5)
h.loglik(z, p, acc)
ts = []
for _ in range(3):
    t0 = time.perf_counter()
    ll = h.loglik(z, p, acc)[0]
    ts.append(time.perf_counter() - t0)
rm = h.rank_map()
np.savez(sys.argv[2], rm=rm, ll=ll)
print(f"acc {acc:g} ll {ll!r} wall {min(ts):.3f} s sum_ranks {rm[rm > 0].sum()}")
