"""MLE driver (f1): same Nelder-Mead trace as the reference's mle_fit
(restated in the oracle), evaluation cap, -inf on NPD.  CPU (injected
objectives); a small device run is marked gpu."""
import math

import numpy as np
import pytest

from oracle import tlr_oracle as orc

BOUNDS = ((0.01, 5.0), (0.001, 3.0), (0.1, 3.0))


def quad_obj(theta):
    t = np.asarray(theta)
    return -float(np.sum(((t - np.array([1.3, 0.2, 0.7])) / np.array([1.0, 0.1, 0.5])) ** 2))


def test_trace_matches_reference_search():
    from paper_1804_09137_b200 import LikelihoodConfig
    from paper_1804_09137_b200.mle import mle_fit
    cfg = LikelihoodConfig(bounds=BOUNDS, max_iterations=40, tol=1e-9)
    res = mle_fit(None, None, cfg, objective=quad_obj)
    x, ll, it, conv, thetas = orc.mle_fit(quad_obj, BOUNDS, max_iterations=40, tol=1e-9)
    assert [e.theta for e in res.trace] == thetas
    assert res.iterations == it and res.converged == conv
    assert res.loglik == pytest.approx(ll, rel=1e-15)


def test_evaluation_cap_and_best_vertex():
    from paper_1804_09137_b200 import LikelihoodConfig
    from paper_1804_09137_b200.mle import mle_fit
    cfg = LikelihoodConfig(bounds=BOUNDS, max_iterations=1000, tol=0.0)
    res = mle_fit(None, None, cfg, objective=quad_obj, max_evaluations=20)
    assert res.evaluations == 20 and len(res.trace) == 20
    best = max(e.loglik for e in res.trace)
    assert res.loglik == best


def test_npd_scores_minus_inf():
    from paper_1804_09137_b200 import LikelihoodConfig
    from paper_1804_09137_b200.mle import mle_fit

    def obj(theta):
        return -math.inf if theta[2] > 1.0 else quad_obj(theta)
    res = mle_fit(None, None, LikelihoodConfig(bounds=BOUNDS, max_iterations=30), objective=obj)
    assert math.isfinite(res.loglik) and res.theta_hat.theta3 <= 1.0


@pytest.mark.gpu
def test_device_mle_small(tb):
    from paper_1804_09137_b200.mle import mle_fit
    locs = tb.generate_locations(400, 0)
    p = tb.MaternParams(1.0, 0.1, 0.5)
    z = tb.sample_measurements(locs, p, 1)
    cfg = tb.LikelihoodConfig(mode="tlr", accuracy=1e-7, nb=100, theta0=(0.8, 0.15, 0.6), max_iterations=200)
    res = mle_fit(locs, z, cfg, max_evaluations=20)
    assert res.evaluations == 20
    ll_true = tb.log_likelihood(locs, z, p, cfg)
    assert res.loglik >= tb.log_likelihood(locs, z, tb.MaternParams(0.8, 0.15, 0.6), cfg)
    assert math.isfinite(ll_true)


@pytest.mark.parametrize("case", ["quad", "quad_theta0", "npd"])
def test_oracle_and_driver_match_reference_traces(case):
    """Pins the oracle restatement and the device driver's search to the
    reference's own mle_fit traces (tests/golden/mle.json)."""
    import json
    from conftest import GOLD
    from paper_1804_09137_b200 import LikelihoodConfig
    from paper_1804_09137_b200.mle import mle_fit
    g = json.loads((GOLD / "mle.json").read_text())[case]
    obj = quad_obj if case != "npd" else (lambda th: -math.inf if th[2] > 1.0 else quad_obj(th))
    kw = g["kw"]
    x, ll, it, conv, thetas = orc.mle_fit(obj, BOUNDS, theta0=kw.get("theta0"),
                                          max_iterations=kw["max_iterations"])
    assert [list(t) for t in thetas] == g["thetas"] and it == g["iterations"] and conv == g["converged"]
    res = mle_fit(None, None, LikelihoodConfig(bounds=BOUNDS, **kw), objective=obj)
    assert [list(e.theta) for e in res.trace] == g["thetas"]
    assert res.loglik == pytest.approx(g["loglik"], rel=1e-15)
