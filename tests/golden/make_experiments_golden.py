"""Golden outputs of the UNMODIFIED reference's accuracy studies
(predict.holdout_experiment, stats.mc_experiment / mc_summaries) on small
seeded cases, for tests/test_experiments.py.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_experiments_golden.py
"""
import json
from pathlib import Path

from tlrgeo import LikelihoodConfig, MaternParams, generate_locations, sample_measurements
from tlrgeo.predict import holdout_experiment
from tlrgeo.stats import mc_experiment, mc_summaries

theta = MaternParams(1.0, 0.1, 0.5)
locs = generate_locations(400, 0)
z = sample_measurements(locs, theta, 1)
ho = holdout_experiment(locs, z, theta, 25, ["dense", "tlr:1e-7"], 2, nb=100)
reps = mc_experiment(150, theta, 3, ["dense", "tlr:1e-7"], 3,
                     LikelihoodConfig(nb=50, max_iterations=12))
out = {"holdout": {"n": 400, "seed_locs": 0, "seed_z": 1, "m": 25, "seed": 2, "nb": 100, "mse": ho},
       "mc": {"n": 150, "replicates": 3, "seed": 3, "nb": 50, "max_iterations": 12,
              "reps": [{"label": r.mode_label, "i": r.replicate,
                        "theta_hat": list(r.result.theta_hat.as_tuple()[:3]) if r.result else None,
                        "loglik": r.result.loglik if r.result else None,
                        "evaluations": len(r.result.trace) if r.result else None} for r in reps],
              "summaries": [{"label": s.mode_label, "medians": list(s.medians), "q1": list(s.q1),
                             "q3": list(s.q3), "failures": s.failures} for s in mc_summaries(reps)]}}
(Path(__file__).resolve().parent / "experiments.json").write_text(json.dumps(out, indent=1))
print(json.dumps(out, indent=1)[:2000])
