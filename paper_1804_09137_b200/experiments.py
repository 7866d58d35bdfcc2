"""Accuracy studies on top of the device path.

Public names follow the reference (`tlrgeo.predict.holdout_experiment` /
`mse`, predict.py:88-127; `tlrgeo.stats.mc_experiment` and its result types,
stats.py:254-339) so that a caller can switch packages; the bodies are this
package's own.  The pieces that must agree with the reference bit for bit are
the seeded draws: the held-out index set (default_rng(seed).choice without
replacement, sorted — predict.py:114-115) and the replicate seeds
(locations `seed`, field `seed + 1 + i` — stats.py:320-327).

Monte Carlo replicates are independent, so under torch.distributed they are
dealt round-robin over the ranks (one GPU each, no collective on the data
path) and gathered once at the end in the reference's (mode, replicate) order.
"""
from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

from .api import (LikelihoodConfig, LocationSet, MaternParams, NotPositiveDefiniteError, PredictionProblem,
                  generate_locations, predict, sample_measurements)
from .mle import EstimationError, EstimationResult, mle_fit

__all__ = ["mse", "parse_mode", "mode_label", "holdout_mask", "holdout_experiment", "empirical_theta0",
           "McReplicate", "McSummary", "mc_summaries", "mc_experiment"]


# ----------------------------------------------------------------- modes
_MODES = ("dense", "tlr")


def parse_mode(spec: str) -> tuple[str, float | None]:
    """Mode spec -> (mode, accuracy): "dense" or "tlr:<eps>", case and
    surrounding blanks ignored (the reference's spec grammar, stats.py:254-263)."""
    name, sep, arg = spec.strip().lower().partition(":")
    if name not in _MODES:
        raise ValueError(f"unknown mode spec {spec!r}")
    if name == "dense":
        if sep:
            raise ValueError(f"unknown mode spec {spec!r}")
        return "dense", None
    if not arg:
        raise ValueError("tlr mode spec needs an accuracy, e.g. tlr:1e-9")
    return "tlr", float(arg)


def mode_label(mode: str, eps: float | None) -> str:
    """Label of a mode as the reference prints it ("dense", "tlr:1e-5"):
    %g of the accuracy with the exponent's leading zero dropped."""
    if mode == "dense":
        return "dense"
    mant, e, exp = f"{eps:g}".partition("e")
    if not e:
        return f"tlr:{mant}"
    sign, digits = exp[0], exp[1:].lstrip("0") or "0"
    return f"tlr:{mant}e{sign}{digits}"


def _as_mode(spec) -> tuple[str, float | None]:
    return parse_mode(spec) if isinstance(spec, str) else (spec[0], spec[1])


# -------------------------------------------------------- hold-out kriging
def mse(truth: np.ndarray, pred: np.ndarray) -> float:
    """Mean squared prediction error over the held-out sites (predict.py:88-97)."""
    t = np.asarray(truth, dtype=float)
    p = np.asarray(pred, dtype=float)
    if t.ndim != 1 or t.shape != p.shape:
        raise ValueError(f"length mismatch: {t.shape} vs {p.shape}")
    r = t - p
    return float(np.dot(r, r)) / r.size


def holdout_mask(n: int, m: int, seed: int) -> np.ndarray:
    """Boolean mask of the m held-out sites: the reference's
    draw default_rng(seed).choice(n, m, replace=False), predict.py:114-115."""
    if not 1 <= m < n:
        raise ValueError(f"need 1 <= m < n, got m={m}, n={n}")
    mask = np.zeros(n, dtype=bool)
    mask[np.random.default_rng(seed).choice(n, size=m, replace=False)] = True
    return mask


def holdout_experiment(locs, z: np.ndarray, theta: MaternParams, m: int, modes, seed: int,
                       nb: int | None = None, max_rank: int | None = None) -> dict[str, float]:
    """Krige the held-out sites from the others in each mode and score the
    MSE, keyed by mode label (predict.holdout_experiment's contract)."""
    z = np.asarray(z, dtype=float)
    held = holdout_mask(len(locs), m, seed)
    metric = getattr(locs, "metric", None)
    known, unknown = LocationSet(locs.coords[~held], metric), LocationSet(locs.coords[held], metric)
    scores = {}
    for spec in modes:
        mode, acc = _as_mode(spec)
        pred = predict(PredictionProblem(known, z[~held], unknown, theta, mode, acc, nb, max_rank=max_rank))
        scores[mode_label(mode, acc)] = mse(z[held], pred)
    return scores


def empirical_theta0(z: np.ndarray, bounds=LikelihoodConfig().bounds) -> tuple:
    """Data-driven simplex start (stats.py:136-141): the sample variance
    (kept strictly inside the theta1 bounds) and the geometric midpoints of
    the range and smoothness bounds."""
    (l1, u1), (l2, u2), (l3, u3) = bounds
    var = min(max(float(np.var(z)), l1 * 1.0001), u1 * 0.9999)
    return (var, float(np.sqrt(l2 * u2)), float(np.sqrt(l3 * u3)))


# ------------------------------------------------------------ Monte Carlo
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
    """Per mode, in first-seen order: median and quartiles of the fitted
    (theta1, theta2, theta3) over the successful replicates, and the number of
    failed ones (stats.py:289-309)."""
    by_label: dict[str, list[McReplicate]] = {}
    for r in replicates:
        by_label.setdefault(r.mode_label, []).append(r)
    out = []
    for label, reps in by_label.items():
        fitted = [r.result.theta_hat.as_tuple()[:3] for r in reps if r.result is not None]
        failed = len(reps) - len(fitted)
        if not fitted:
            out.append(McSummary(label, (), (), (), failed))
            continue
        q = np.percentile(np.asarray(fitted), [25, 50, 75], axis=0)
        out.append(McSummary(label, tuple(q[1]), tuple(q[0]), tuple(q[2]), failed))
    return out


def _torch_dist():
    try:
        import torch.distributed as dist
    except ImportError:
        return None
    return dist if dist.is_available() and dist.is_initialized() else None


def mc_experiment(n: int, theta_true: MaternParams, replicates: int, modes, seed: int,
                  cfg: LikelihoodConfig = LikelihoodConfig(), empirical_start: bool = True,
                  fit=None, sampler=None) -> list[McReplicate]:
    """Parameter-recovery study (stats.mc_experiment's contract): one
    location set from `seed`; replicate i is measured with seed + 1 + i and
    fitted in every mode; a failed fit is recorded, not raised.  The result
    list is ordered by (mode, replicate) on every rank.  `fit(locs, z, cfg)`
    and `sampler(locs, theta, seed)` default to the device mle_fit /
    sample_measurements (host-side tests inject CPU stand-ins)."""
    fit = fit or mle_fit
    sampler = sampler or sample_measurements
    locs = generate_locations(n, seed)
    dist = _torch_dist()
    rank, world = (dist.get_rank(), dist.get_world_size()) if dist else (0, 1)
    specs = [_as_mode(s) for s in modes]
    mine = range(rank, replicates, world)
    fields = {i: sampler(locs, theta_true, seed + 1 + i) for i in mine}
    done: dict[tuple[int, int], McReplicate] = {}
    for mi, (mode, acc) in enumerate(specs):
        label = mode_label(mode, acc)
        base = replace(cfg, mode=mode, accuracy=acc)
        for i in mine:
            run = base
            if empirical_start and run.theta0 is None:
                run = replace(run, theta0=empirical_theta0(fields[i], cfg.bounds))
            try:
                done[(mi, i)] = McReplicate(label, i, fit(locs, fields[i], run))
            except (EstimationError, NotPositiveDefiniteError) as exc:
                done[(mi, i)] = McReplicate(label, i, None, str(exc))
    if dist and world > 1:
        parts = [None] * world
        dist.all_gather_object(parts, done)
        done = {k: v for part in parts for k, v in part.items()}
    return [done[k] for k in sorted(done)]
