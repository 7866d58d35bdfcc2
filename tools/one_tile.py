"""Compress one C2 offset-1 tile (500x500, acc 1e-9) on the device: isolates
the per-matrix cost of the compressor kernels for ncu."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_1804_09137_b200 as tb
from paper_1804_09137_b200 import _lib

ACC = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-9
locs = tb.generate_locations(10000, 0)
xy = locs.coords
a = tb.matern_block(xy[500:1000], xy[0:500], tb.MaternParams(1.0, 0.1, 0.5))
u, v = tb.compress_tile(a, ACC)
_lib.profile_enable(True)
t0 = time.perf_counter()
u, v = tb.compress_tile(a, ACC)
dt = time.perf_counter() - t0
prof = _lib.profile_read()
print("rank", u.shape[1], "err", np.linalg.norm(a - u @ v.T) / np.linalg.norm(a), f"wall {dt*1e3:.1f} ms")
for k, d in prof.items():
    if d["launches"]:
        print(f"  {k:16s} {d['ms']:8.2f} ms  {d['flops']/1e9:8.2f} GF  launches {d['launches']}")
