"""C3p kriging golden from the UNMODIFIED reference: the C3
patch (generate_locations(62500, 0) restricted to x, y < 0.4, n = 10,000,
z = sample_measurements(patch, theta, 1) as in make_patch_goldens.py), 50
held-out sites drawn like predict.holdout_experiment (default_rng(2)), and
the reference's predict() in dense mode and TLR(1e-9) / TLR(1e-7) at
nb = 760.  Writes tests/golden/c3p_kriging.npz (~5 min of CPU).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_c3p_kriging_golden.py
"""
import time
from pathlib import Path

import numpy as np

from tlrgeo import LocationSet, MaternParams, PredictionProblem, generate_locations, predict

OUT = Path(__file__).resolve().parent
full = generate_locations(62_500, 0).coords
sel = (full[:, 0] < 0.4) & (full[:, 1] < 0.4)
locs = LocationSet(full[sel])
z = np.load(OUT / "z_patches.npz")["C3p"]
p = MaternParams(1.0, 0.03, 0.5)
n = len(locs)
rng = np.random.default_rng(2)
idx = np.sort(rng.choice(n, size=50, replace=False))
mask = np.zeros(n, bool)
mask[idx] = True
known, unknown = LocationSet(locs.coords[~mask]), LocationSet(locs.coords[mask])
out = {"idx": idx}
for key, mode, acc in (("dense", "dense", None), ("tlr_1e-9", "tlr", 1e-9), ("tlr_1e-7", "tlr", 1e-7)):
    t0 = time.time()
    out[key] = predict(PredictionProblem(known, z[~mask], unknown, p, mode, acc, 760))
    print(key, time.time() - t0, flush=True)
np.savez(OUT / "c3p_kriging.npz", **out)
