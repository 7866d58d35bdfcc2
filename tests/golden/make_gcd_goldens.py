"""Great-circle (haversine) metric goldens from the UNMODIFIED reference:
tile (exact evaluator), dense / TLR log-likelihoods and kriging on lon/lat
points (kernels.py:460-491, geometry.py:41-48,106-122).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_gcd_goldens.py
"""
import json
from pathlib import Path

import numpy as np

from tlrgeo import (GreatCircle, LikelihoodConfig, LocationSet, MaternParams, PredictionProblem,
                    assemble_covariance, TileGrid, log_likelihood, predict, sample_measurements)

OUT = Path(__file__).resolve().parent
rng = np.random.default_rng(11)
n = 600
coords = np.column_stack((rng.uniform(38.0, 52.0, n), rng.uniform(14.0, 30.0, n)))   # lon, lat degrees
locs = LocationSet(coords, GreatCircle())
theta = MaternParams(1.0, 300.0, 0.5)                                                 # range in km
tile = assemble_covariance(LocationSet(coords[:64], GreatCircle()), theta, TileGrid(64, 64), "dense",
                           profile="never").diag[0]
z = sample_measurements(locs, theta, 1)
res = {"n": n, "theta": [1.0, 300.0, 0.5], "nb": 150, "modes": {}}
for mode, acc in [("dense", None), ("tlr", 1e-7), ("tlr", 1e-9)]:
    cfg = LikelihoodConfig(mode=mode, accuracy=acc, nb=150)
    res["modes"]["dense" if acc is None else f"tlr:{acc:g}"] = {"ll": log_likelihood(locs, z, theta, cfg)}
known = LocationSet(coords[:560], GreatCircle())
unknown = LocationSet(coords[560:], GreatCircle())
pred = predict(PredictionProblem(known, z[:560], unknown, theta, "dense", None, 150))
np.savez(OUT / "gcd.npz", coords=coords, tile=tile, z=z, pred=pred)
(OUT / "gcd.json").write_text(json.dumps(res, indent=1))
print(res)
