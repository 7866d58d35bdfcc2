"""One warm C2 TLR evaluation (acc from argv, default 1e-9) for TLRB_TRACE runs:
    TLRB_TRACE=1 python tools/trace_c2.py 1e-9 2> trace.log"""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1804_09137_b200 as tb  # noqa: E402

acc = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-9
locs = tb.generate_locations(10000, 0)
z = np.load(Path(__file__).resolve().parents[1] / "tests/golden/z_big.npz")["C2"]
h = tb.Handle(locs.coords, 500)
p = tb.MaternParams(1.0, 0.1, 0.5)
h.loglik(z, p, acc)
print("---- warm", file=sys.stderr, flush=True)
t0 = time.perf_counter()
ll = h.loglik(z, p, acc)
print(f"ll {ll[0]!r}  wall {time.perf_counter() - t0:.3f} s  stats {h.last_stats}")
