"""Compress small tiles of increasing size (debugging aid for the Jacobi kernel)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_1804_09137_b200 as tb
xy = tb.generate_locations(10000, 0).coords
for m in [int(a) for a in sys.argv[1:]]:
    a = tb.matern_block(xy[m:2 * m], xy[0:m], tb.MaternParams(1.0, 0.1, 0.5))
    t0 = time.time()
    u, v = tb.compress_tile(a, 1e-9)
    print(m, "rank", u.shape[1], "err", np.linalg.norm(a - u @ v.T) / np.linalg.norm(a), f"{time.time()-t0:.3f}s", flush=True)
