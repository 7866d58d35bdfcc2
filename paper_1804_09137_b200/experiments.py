"""Accuracy studies on top of the device path: the hold-out
kriging MSE driver (predict.py:88-127) and the Monte Carlo parameter-recovery
study (stats.py:254-339), with the reference's names, seeds and result
types.  Replicates of `mc_experiment` run as independent replicas across the
GPUs of a torch.distributed job (replicate i on rank i mod world, results
all-gathered); every likelihood evaluation is the CUDA path of `mle_fit`.
"""
from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

from .api import (LikelihoodConfig, LocationSet, MaternParams, NotPositiveDefiniteError, PredictionProblem,
                  generate_locations, predict, sample_measurements)
from .mle import EstimationError, EstimationResult, mle_fit

__all__ = ["mse", "parse_mode", "mode_label", "holdout_experiment", "empirical_theta0", "McReplicate",
           "McSummary", "mc_summaries", "mc_experiment"]


def mse(truth: np.ndarray, pred: np.ndarray) -> float:
    """Mean squared error (1/m) sum (Y_i - Yhat_i)^2 (predict.py:88-97)."""
    truth = np.asarray(truth, dtype=float)
    pred = np.asarray(pred, dtype=float)
    if truth.shape != pred.shape or truth.ndim != 1:
        raise ValueError(f"length mismatch: {truth.shape} vs {pred.shape}")
    d = truth - pred
    return float(d @ d) / truth.size


def parse_mode(spec: str) -> tuple[str, float | None]:
    """"dense" or "tlr:EPS" (stats.py:254-263)."""
    spec = spec.strip().lower()
    if spec == "dense":
        return "dense", None
    if spec.startswith("tlr:"):
        return "tlr", float(spec.split(":", 1)[1])
    if spec == "tlr":
        raise ValueError("tlr mode spec needs an accuracy, e.g. tlr:1e-9")
    raise ValueError(f"unknown mode spec {spec!r}")


def mode_label(mode: str, eps: float | None) -> str:
    """Canonical label, e.g. "dense" or "tlr:1e-5" (stats.py:266-270)."""
    if mode == "dense":
        return "dense"
    return "tlr:" + f"{eps:g}".replace("e-0", "e-").replace("e+0", "e+")


def holdout_experiment(locs, z: np.ndarray, theta: MaternParams, m: int, modes, seed: int,
                       nb: int | None = None, max_rank: int | None = None) -> dict[str, float]:
    """Hold out m sites drawn without replacement (default_rng(seed)), krige
    them from the rest in every mode, score the MSE (predict.py:100-127)."""
    n = len(locs)
    z = np.asarray(z, dtype=float)
    if not 1 <= m < n:
        raise ValueError(f"need 1 <= m < n, got m={m}, n={n}")
    rng = np.random.default_rng(seed)
    unknown_idx = np.sort(rng.choice(n, size=m, replace=False))
    mask = np.zeros(n, dtype=bool)
    mask[unknown_idx] = True
    metric = getattr(locs, "metric", None)
    known = LocationSet(locs.coords[~mask], metric)
    unknown = LocationSet(locs.coords[mask], metric)
    out = {}
    for spec in modes:
        mode, acc = parse_mode(spec) if isinstance(spec, str) else spec
        problem = PredictionProblem(known, z[~mask], unknown, theta, mode, acc, nb, max_rank=max_rank)
        out[mode_label(mode, acc)] = mse(z[mask], predict(problem))
    return out


def empirical_theta0(z: np.ndarray, bounds=LikelihoodConfig().bounds) -> tuple:
    """Variance-matched start: var(z) for theta1, log-midpoints of the
    bounds for range and smoothness (stats.py:136-141)."""
    (l1, u1), (l2, u2), (l3, u3) = bounds
    v = float(np.clip(np.var(z), l1 * 1.0001, u1 * 0.9999))
    return (v, float(np.sqrt(l2 * u2)), float(np.sqrt(l3 * u3)))


@dataclass
class McReplicate:
    mode_label: str
    replicate: int
    result: EstimationResult | None
    error: str | None = None


@dataclass
class McSummary:
    mode_label: str
    medians: tuple
    q1: tuple
    q3: tuple
    failures: int


def mc_summaries(replicates: list[McReplicate]) -> list[McSummary]:
    """Per mode: median and quartiles of theta_hat, failure count (stats.py:289-309)."""
    out = []
    for label in dict.fromkeys(r.mode_label for r in replicates):
        thetas = np.array([r.result.theta_hat.as_tuple()[:3]
                           for r in replicates if r.mode_label == label and r.result is not None])
        failures = sum(1 for r in replicates if r.mode_label == label and r.result is None)
        if thetas.size:
            out.append(McSummary(label, tuple(np.median(thetas, axis=0)), tuple(np.percentile(thetas, 25, axis=0)),
                                 tuple(np.percentile(thetas, 75, axis=0)), failures))
        else:
            out.append(McSummary(label, (), (), (), failures))
    return out


def _dist():
    try:
        import torch.distributed as dist
    except ImportError:
        return None
    return dist if dist.is_available() and dist.is_initialized() else None


def mc_experiment(n: int, theta_true: MaternParams, replicates: int, modes, seed: int,
                  cfg: LikelihoodConfig = LikelihoodConfig(), empirical_start: bool = True,
                  fit=None, sampler=None) -> list[McReplicate]:
    """Monte Carlo recovery study (stats.py:312-339): one location set from
    `seed`, replicate i measured with seed + 1 + i, every mode fitted to every
    replicate; failures are recorded, not fatal.  Under torch.distributed the
    replicates are independent replicas spread over the ranks (one GPU each)
    and every rank returns the full list in the reference's order.
    `fit(locs, z, cfg)` / `sampler(locs, theta, seed)` default to the device
    `mle_fit` / `sample_measurements` (hooks for host-side tests)."""
    fit = fit or mle_fit
    sampler = sampler or sample_measurements
    locs = generate_locations(n, seed)
    d = _dist()
    rank, world = (d.get_rank(), d.get_world_size()) if d else (0, 1)
    mine = [i for i in range(replicates) if i % world == rank]
    zs = {i: sampler(locs, theta_true, seed + 1 + i) for i in mine}
    local: list[tuple[int, int, McReplicate]] = []
    for mi, spec in enumerate(modes):
        mode, acc = parse_mode(spec) if isinstance(spec, str) else spec
        label = mode_label(mode, acc)
        for i in mine:
            run_cfg = replace(cfg, mode=mode, accuracy=acc)
            if empirical_start and run_cfg.theta0 is None:
                run_cfg = replace(run_cfg, theta0=empirical_theta0(zs[i], cfg.bounds))
            try:
                local.append((mi, i, McReplicate(label, i, fit(locs, zs[i], run_cfg))))
            except (EstimationError, NotPositiveDefiniteError) as exc:
                local.append((mi, i, McReplicate(label, i, None, str(exc))))
    if d and world > 1:
        parts = [None] * world
        d.all_gather_object(parts, local)
        local = [x for part in parts for x in part]
    return [r for _, _, r in sorted(local, key=lambda t: (t[0], t[1]))]
