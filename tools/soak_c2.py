"""Soak test: many C2 TLR evaluations on one handle at varying theta (the MLE
access pattern) — device memory, time per evaluation and bitwise repeatability.
    python tools/soak_c2.py [evals]"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1804_09137_b200 as tb  # noqa: E402

nev = int(sys.argv[1]) if len(sys.argv) > 1 else 30
locs = tb.generate_locations(10000, 0)
z = np.load(Path(__file__).resolve().parents[1] / "tests/golden/z_big.npz")["C2"]
h = tb.Handle(locs.coords, 500)
rng = np.random.default_rng(0)
first = None
free0 = torch.cuda.mem_get_info()[0]
ts = []
for e in range(nev):
    th = (1.0, 0.1, 0.5) if e % 5 == 0 else (rng.uniform(0.5, 2), rng.uniform(0.03, 0.3), rng.uniform(0.3, 1.5))
    t0 = time.perf_counter()
    ll = h.loglik(z, tb.MaternParams(*th), 1e-9)[0]
    ts.append(time.perf_counter() - t0)
    if e % 5 == 0:
        if first is None:
            first = ll
        assert ll == first, (e, ll, first)
free1 = torch.cuda.mem_get_info()[0]
print(f"evals {nev}  median {np.median(ts):.3f} s  max {max(ts):.3f} s  repeat-ll identical  "
      f"free-memory drift {(free0 - free1) / 2**20:.1f} MiB")
