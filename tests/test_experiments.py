"""Accuracy studies: hold-out kriging MSE driver and the
Monte Carlo recovery study, against the unmodified reference's outputs
(tests/golden/make_experiments_golden.py).  Host logic and the replica
sharding over ranks run on CPU with the oracle as the likelihood; the
device path is marked gpu."""
import json
import math
import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import GOLD
from oracle import tlr_oracle as orc
from paper_1804_09137_b200 import LikelihoodConfig, LocationSet, MaternParams
from paper_1804_09137_b200 import experiments as ex
from paper_1804_09137_b200.mle import EstimationError, mle_fit

G = json.loads((GOLD / "experiments.json").read_text())
THETA = MaternParams(1.0, 0.1, 0.5)


def test_mse_and_mode_labels():
    assert ex.mse(np.array([1.0, 2.0, 3.0]), np.array([1.0, 0.0, 3.0])) == pytest.approx(4.0 / 3.0)
    with pytest.raises(ValueError):
        ex.mse(np.zeros(3), np.zeros(2))
    assert ex.parse_mode("dense") == ("dense", None)
    assert ex.parse_mode(" TLR:1e-9 ") == ("tlr", 1e-9)
    with pytest.raises(ValueError):
        ex.parse_mode("tlr")
    with pytest.raises(ValueError):
        ex.parse_mode("hodlr:1e-3")
    assert ex.mode_label("tlr", 1e-5) == "tlr:1e-5" and ex.mode_label("dense", None) == "dense"
    assert ex.mode_label("tlr", 2.5e-10) == "tlr:2.5e-10"
    assert [s["label"] for s in G["mc"]["summaries"]] == ["dense", "tlr:1e-7"]


def test_empirical_theta0():
    z = np.random.default_rng(0).standard_normal(500) * 2.0
    b = LikelihoodConfig().bounds
    t = ex.empirical_theta0(z, b)
    assert t[0] == pytest.approx(np.var(z)) and t[1] == pytest.approx(math.sqrt(0.001 * 3.0))
    assert ex.empirical_theta0(np.zeros(4), b)[0] == pytest.approx(0.01 * 1.0001)


def test_estimation_error_contract():
    with pytest.raises(EstimationError) as e:
        mle_fit(None, None, LikelihoodConfig(max_iterations=3), objective=lambda th: -math.inf)
    assert "no likelihood evaluation succeeded; last theta tried" in str(e.value)
    assert len(e.value.last_theta) == 3


def _oracle_fit(locs, z, cfg):
    acc = cfg.accuracy if cfg.mode == "tlr" else None
    return mle_fit(locs, z, cfg, objective=lambda th: orc.log_likelihood(locs.coords, z, tuple(th), cfg.nb, acc)[0])


def _oracle_sampler(locs, theta, seed):
    return orc.sample_measurements(locs.coords, theta.as_tuple()[:3], seed)


def _mc_cfg():
    g = G["mc"]
    return LikelihoodConfig(nb=g["nb"], max_iterations=g["max_iterations"])


def _check_mc(reps):
    g = G["mc"]
    assert [(r.mode_label, r.replicate) for r in reps] == [(x["label"], x["i"]) for x in g["reps"]]
    for r, x in zip(reps, g["reps"]):
        assert r.result is not None
        np.testing.assert_allclose(r.result.theta_hat.as_tuple()[:3], x["theta_hat"], rtol=1e-7)
        assert r.result.evaluations == x["evaluations"]
    for s, x in zip(ex.mc_summaries(reps), g["summaries"]):
        assert s.failures == x["failures"]
        np.testing.assert_allclose(s.medians, x["medians"], rtol=1e-7)
        np.testing.assert_allclose(s.q1, x["q1"], rtol=1e-7)


def test_mc_experiment_host_logic_matches_reference():
    """Seeds, replicate order, empirical start, summaries: the reference's
    mc_experiment output with the oracle as the likelihood."""
    g = G["mc"]
    reps = ex.mc_experiment(g["n"], THETA, g["replicates"], ["dense", "tlr:1e-7"], g["seed"], _mc_cfg(),
                            fit=_oracle_fit, sampler=_oracle_sampler)
    _check_mc(reps)


def _mc_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = G["mc"]
        reps = ex.mc_experiment(g["n"], THETA, g["replicates"], ["dense", "tlr:1e-7"], g["seed"], _mc_cfg(),
                                fit=_oracle_fit, sampler=_oracle_sampler)
        out[rank] = [(r.mode_label, r.replicate, r.result.theta_hat.as_tuple()[:3]) for r in reps]
    finally:
        dist.destroy_process_group()


def test_mc_replicas_across_ranks():
    """Replicates spread over 2 ranks (gloo): every rank gets the full,
    ordered list, equal to the reference's."""
    port = 29500 + os.getpid() % 2000
    out = mp.Manager().dict()
    mp.spawn(_mc_worker, args=(2, port, out), nprocs=2, join=True)
    g = G["mc"]
    want = [(x["label"], x["i"]) for x in g["reps"]]
    for rank in (0, 1):
        assert [(a, b) for a, b, _ in out[rank]] == want
        for (_, _, th), x in zip(out[rank], g["reps"]):
            np.testing.assert_allclose(th, x["theta_hat"], rtol=1e-7)


@pytest.mark.gpu
def test_holdout_experiment_device(tb):
    g = G["holdout"]
    locs = tb.generate_locations(g["n"], g["seed_locs"])
    z = orc.sample_measurements(locs.coords, (1.0, 0.1, 0.5), g["seed_z"])   # = the reference's z
    got = ex.holdout_experiment(locs, z, THETA, g["m"], ["dense", "tlr:1e-7"], g["seed"], nb=g["nb"])
    assert got["dense"] == pytest.approx(g["mse"]["dense"], rel=1e-10)
    assert got["tlr:1e-7"] == pytest.approx(g["mse"]["tlr:1e-7"], rel=1e-6)


@pytest.mark.gpu
def test_mc_experiment_device(tb):
    g = G["mc"]
    reps = ex.mc_experiment(g["n"], THETA, g["replicates"], ["dense", "tlr:1e-7"], g["seed"], _mc_cfg())
    _check_mc(reps)
