"""Kriging conditional-variance golden (predict.py:81-87, dense mode only)
from the UNMODIFIED reference.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_variance_golden.py
"""
from pathlib import Path

import numpy as np

from tlrgeo import LocationSet, MaternParams, PredictionProblem, generate_locations, predict, sample_measurements

theta = MaternParams(1.0, 0.1, 0.5, 0.01)
locs = generate_locations(320, 4)
z = sample_measurements(locs, theta, 5)
known = LocationSet(locs.coords[:300])
unknown = LocationSet(locs.coords[300:])
pred, cov = predict(PredictionProblem(known, z[:300], unknown, theta, nb=100), with_variance=True)
np.savez(Path(__file__).resolve().parent / "variance.npz", known=known.coords, unknown=unknown.coords,
         z=z[:300], pred=pred, cov=cov)
print(pred[:3], np.diag(cov)[:3])
