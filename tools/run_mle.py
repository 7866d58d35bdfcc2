"""MLE at a BASELINE config on one GPU: z from the device
sampler (stats.py:115-133 semantics), the reference's empirical start
(stats.py:136-141), bounded Nelder-Mead capped at 20 likelihood evaluations
(the C5 protocol, run here at C2 / C3 size), then kriging of m held-out
sites with theta_hat (predict.holdout_experiment index draw).

    python tools/run_mle.py C3 [--evals 20]
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1804_09137_b200 as tb  # noqa: E402
from paper_1804_09137_b200.experiments import empirical_theta0, mse  # noqa: E402
from tools.run_config import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--evals", type=int, default=20)
    a = ap.parse_args()
    c = CONFIGS[a.config]
    locs = tb.generate_locations(c["n"], 0)
    p_true = tb.MaternParams(*c["theta"])
    z = tb.sample_measurements(locs, p_true, 1)
    m = c["m"] or 100
    rng = np.random.default_rng(2)
    idx = np.sort(rng.choice(c["n"], size=m, replace=False))
    mask = np.zeros(c["n"], bool)
    mask[idx] = True
    known, unknown = tb.LocationSet(locs.coords[~mask]), tb.LocationSet(locs.coords[mask])
    cfg = tb.LikelihoodConfig(mode="tlr", accuracy=c["acc"], nb=c["nb"], max_rank=c["max_rank"],
                              theta0=empirical_theta0(z[~mask]))
    t0 = time.perf_counter()
    res = tb.mle_fit(known, z[~mask], cfg, max_evaluations=a.evals)
    t_mle = time.perf_counter() - t0
    t0 = time.perf_counter()
    pred = tb.predict(tb.PredictionProblem(known, z[~mask], unknown, res.theta_hat, "tlr", c["acc"], c["nb"],
                                           max_rank=c["max_rank"]))
    t_kr = time.perf_counter() - t0
    secs = [e.seconds for e in res.trace]
    print(json.dumps({"config": a.config, "n_known": int((~mask).sum()), "m": m, "theta_true": c["theta"],
                      "theta0": list(cfg.theta0), "theta_hat": list(res.theta_hat.as_tuple()[:3]),
                      "loglik": res.loglik, "evaluations": res.evaluations, "mle_s": t_mle,
                      "eval_s_median": float(np.median(secs)), "eval_s_first": secs[0],
                      "kriging_s": t_kr, "kriging_mse": mse(z[mask], pred),
                      "trace": [[list(e.theta), e.loglik] for e in res.trace]}))


if __name__ == "__main__":
    main()
