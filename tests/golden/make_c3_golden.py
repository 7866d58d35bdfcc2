"""Full C3 golden from the UNMODIFIED reference (slow: ~15 min, ~32 GB RAM):
z = sample_measurements(generate_locations(62500, 0), (1, 0.03, 0.5), 1) and the
dense log-likelihood at nb = 760.  The C3 TLR(1e-7)
reference (~5 h) is not generated.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_c3_golden.py
"""
import json
import math
import time
from pathlib import Path

import numpy as np

from tlrgeo import MaternParams, TileGrid, assemble_covariance, generate_locations, sample_measurements
from tlrgeo import linalg

OUT = Path(__file__).resolve().parent
locs = generate_locations(62_500, 0)
p = MaternParams(1.0, 0.03, 0.5)
t0 = time.time()
z = sample_measurements(locs, p, 1)
np.savez_compressed(OUT / "z_c3.npz", C3=z)
print("z", time.time() - t0, flush=True)
t1 = time.time()
cov = assemble_covariance(locs, p, TileGrid(62_500, 760), "dense")
f = linalg.cholesky(cov)
quad = linalg.quadratic_form(f, z)
ll = -0.5 * (62_500 * math.log(2 * math.pi) + f.log_det + quad)
(OUT / "c3.json").write_text(json.dumps({"C3": {"n": 62500, "theta": [1.0, 0.03, 0.5], "nb": 760,
                                                "modes": {"dense": {"ll": ll, "log_det": f.log_det,
                                                                    "quad": quad,
                                                                    "seconds": time.time() - t1}}}},
                                        indent=1))
print("dense", ll, time.time() - t1, flush=True)
