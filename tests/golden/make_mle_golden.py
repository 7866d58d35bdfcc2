"""Golden Nelder-Mead traces from the UNMODIFIED reference stats.mle_fit with
injected objectives (its objective= hook, stats.py:167-168).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_mle_golden.py
"""
import json
import math
from pathlib import Path

import numpy as np

from tlrgeo import LikelihoodConfig, mle_fit

BOUNDS = ((0.01, 5.0), (0.001, 3.0), (0.1, 3.0))


def quad_obj(theta):
    t = np.asarray(theta)
    return -float(np.sum(((t - np.array([1.3, 0.2, 0.7])) / np.array([1.0, 0.1, 0.5])) ** 2))


def npd_obj(theta):
    return -math.inf if theta[2] > 1.0 else quad_obj(theta)


out = {}
for name, obj, kw in [("quad", quad_obj, dict(max_iterations=40)),
                      ("quad_theta0", quad_obj, dict(max_iterations=25, theta0=(4.5, 2.5, 0.2))),
                      ("npd", npd_obj, dict(max_iterations=30))]:
    res = mle_fit(None, None, LikelihoodConfig(bounds=BOUNDS, **kw), objective=obj)
    out[name] = {"kw": {k: v for k, v in kw.items()}, "thetas": [list(e.theta) for e in res.trace],
                 "iterations": res.iterations, "converged": res.converged, "loglik": res.loglik,
                 "theta_hat": list(res.theta_hat.as_tuple()[:3])}
(Path(__file__).resolve().parent / "mle.json").write_text(json.dumps(out, indent=1))
print({k: (len(v["thetas"]), v["iterations"], v["converged"]) for k, v in out.items()})
