"""Maximum-likelihood driver on a persistent device handle.

Same search as the reference's `stats.mle_fit` (stats.py:144-251): bounded
Nelder-Mead over (theta1, theta2, theta3) with coefficients
(reflect, expand, contract, shrink) = (1, 2, 1/2, 1/2), out-of-bounds
proposals clamped, initial simplex of +25% steps flipped at the upper bound,
stop when the relative objective spread <= tol or after max_iterations, and
a not-positive-definite evaluation scoring -inf.  Added for the C5 config:
`max_evaluations` stops after that many objective calls and returns the best
vertex seen.  Every evaluation runs on the GPU through one Handle, so the
locations and tile arenas stay resident across the whole search.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

from .api import LikelihoodConfig, MaternParams, NotPositiveDefiniteError, _coords_of, _handle_for, _radius_of


@dataclass(frozen=True)
class TraceEntry:
    index: int
    theta: tuple
    loglik: float
    seconds: float


@dataclass
class EstimationResult:
    """stats.py:82-93 (+ `evaluations`, the objective calls made)."""

    theta_hat: MaternParams
    loglik: float
    iterations: int
    converged: bool
    evaluations: int
    trace: list = field(repr=False, default_factory=list)
    mode: str = "dense"
    accuracy: float | None = None

    @property
    def total_seconds(self) -> float:
        return sum(t.seconds for t in self.trace)


class EstimationError(Exception):
    """Every objective evaluation failed (stats.py:31-38): same message and
    `last_theta` attribute as the reference."""

    def __init__(self, last_theta):
        self.last_theta = tuple(last_theta)
        super().__init__(
            f"no likelihood evaluation succeeded; last theta tried {self.last_theta}"
        )


class _Budget(Exception):
    pass


def _start(x0, bounds):
    """Initial simplex: x0 plus one +25% step per coordinate, flipped (and
    clamped) at the upper bound (stats.py:148-158)."""
    pts = [x0.copy()]
    for d, (lo, hi) in enumerate(bounds):
        step = 0.25 * x0[d]
        if x0[d] + step > hi:
            step = -step
        v = x0.copy()
        v[d] = min(max(v[d] + step, lo), hi)
        pts.append(v)
    return pts


def mle_fit(locs, z, cfg: LikelihoodConfig, objective=None, max_evaluations: int | None = None):
    bounds = cfg.bounds
    lo = np.array([b[0] for b in bounds])
    hi = np.array([b[1] for b in bounds])
    if objective is None:
        coords = _coords_of(locs)
        h = _handle_for(coords, min(cfg.tile_size(), len(locs)), cfg.max_rank, cfg.ngpus, _radius_of(locs))
        acc = cfg.accuracy if cfg.mode == "tlr" else None
        zz = np.ascontiguousarray(z, dtype=float)

        def objective(theta):
            try:
                return h.loglik(zz, MaternParams(theta[0], theta[1], theta[2], cfg.nugget), acc)[0]
            except NotPositiveDefiniteError:
                return -math.inf

    trace: list[TraceEntry] = []
    best = {"f": math.inf, "x": None}

    def f(x):
        if max_evaluations is not None and len(trace) >= max_evaluations:
            raise _Budget()
        t0 = time.perf_counter()
        ll = objective(x)
        trace.append(TraceEntry(len(trace), tuple(float(v) for v in x), ll, time.perf_counter() - t0))
        val = -ll if math.isfinite(ll) else math.inf
        if val < best["f"]:
            best["f"], best["x"] = val, x.copy()
        return val

    def clip(x):
        return np.minimum(np.maximum(x, lo), hi)

    x0 = np.asarray(cfg.theta0 if cfg.theta0 is not None else np.sqrt(lo * hi), dtype=float)
    x0 = clip(x0)
    pts, vals = [], []
    it, converged = 0, False
    try:
        pts = _start(x0, bounds)
        vals = [f(p) for p in pts]
        while it < cfg.max_iterations:
            order = np.argsort(vals, kind="stable")
            pts = [pts[k] for k in order]
            vals = [vals[k] for k in order]
            fb, fw = vals[0], vals[-1]
            spread = (math.inf if not (math.isfinite(fb) and math.isfinite(fw))
                      else 2.0 * abs(fw - fb) / (abs(fw) + abs(fb) + 1e-300))
            if spread <= cfg.tol:
                converged = True
                break
            it += 1
            cen = np.mean(pts[:-1], axis=0)
            xr = clip(cen + (cen - pts[-1]))
            fr = f(xr)
            if vals[0] <= fr < vals[-2]:
                pts[-1], vals[-1] = xr, fr
            elif fr < vals[0]:
                xe = clip(cen + 2.0 * (xr - cen))
                fe = f(xe)
                pts[-1], vals[-1] = (xe, fe) if fe < fr else (xr, fr)
            else:
                xc = clip(cen + 0.5 * ((xr if fr < vals[-1] else pts[-1]) - cen))
                fc = f(xc)
                if fc < min(fr, vals[-1]):
                    pts[-1], vals[-1] = xc, fc
                else:
                    for q in range(1, len(pts)):
                        pts[q] = clip(pts[0] + 0.5 * (pts[q] - pts[0]))
                        vals[q] = f(pts[q])
    except _Budget:
        pass
    if best["x"] is None or not math.isfinite(best["f"]):
        # the reference reports the simplex's best vertex (stats.py:238-240)
        if len(vals) == len(pts) and pts:
            last = tuple(float(v) for v in pts[int(np.argmin(vals))])
        else:
            last = tuple(float(v) for v in x0)
        raise EstimationError(last)
    x = best["x"]
    return EstimationResult(MaternParams(x[0], x[1], x[2], cfg.nugget), -best["f"], it, converged,
                            len(trace), trace, mode=cfg.mode, accuracy=cfg.accuracy)
