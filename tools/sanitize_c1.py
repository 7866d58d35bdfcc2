"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
C1-sized dense and TLR evaluations (cluster QRCP, cluster Jacobi with DSMEM,
mbarriers and named barriers; blocked randomized QRCP when
TLRB_QRCP_BLOCKED=1), a factored recompression case (nb = 760 patch
geometry, small n), solves, kriging and a 2-rank loopback group handle.

    compute-sanitizer --tool racecheck python tools/sanitize_c1.py
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1804_09137_b200 as tb  # noqa: E402

locs = tb.generate_locations(1600, 0)
z = np.random.default_rng(1).standard_normal(1600)
p = tb.MaternParams(1.0, 0.1, 0.5)
h = tb.Handle(locs.coords, 400)
for acc in (None, 1e-9, 1e-5):
    print("C1", acc, h.loglik(z, p, acc)[0], flush=True)
print("solve", float(np.linalg.norm(h.solve(z))), flush=True)
print("predict", h.predict(z, np.array([[0.5, 0.5], [0.1, 0.9]]), p, 1e-9), flush=True)
h.close()
big = tb.generate_locations(2280, 3)                       # 3 tiles of 760: nb > 512 kernels
hb = tb.Handle(big.coords, 760, max_rank=200)
print("nb760", hb.loglik(np.ones(2280), tb.MaternParams(1.0, 0.03, 0.5), 1e-7)[0], flush=True)
hb.close()
g = tb.group_handle(locs.coords, 400, 2)
print("group", g.loglik(z, p, 1e-9)[0], flush=True)
g.close()
