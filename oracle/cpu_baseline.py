"""Bounded-sample CPU timing of the oracle port (test / bench infrastructure).

Used only by bench.py's `cpu_baseline` leg and `--impl reference` arm.  A full
TLR evaluation of the CPU path at C2 takes minutes (SURVEY.md section 6:
104-214 s on 8 cores), so one "step" times a stratified sample of the
evaluation's work units with the same oracle code and extrapolates by exact
unit counts:

  * tile generation + compression: one tile per tile offset d = i - j
    (cost x (t - d) tiles)                        [tilestore.py:181-223]
  * POTRF of one diagonal tile (x t), TRSM and SYRK of one panel tile
    (x t(t-1)/2 each)                             [linalg.py:117-132]
  * GEMM + recompression for sampled offset pairs (d1 = i - j, d2 = j - k),
    cost interpolated in the stacked rank K = k_ij + k_jk and weighted by the
    (t - d1 - d2) triples per pair                [linalg.py:133-139]
  * forward solve over all stored tiles           [linalg.py:166-177]

The dense mode runs the whole oracle evaluation (seconds at C2).
"""
from __future__ import annotations

import os
import time

import numpy as np
import scipy.linalg as sla

from . import tlr_oracle as orc


def _t(fn, *a, reps: int = 2):
    """Best of `reps` timings (the first call of a shape can carry LAPACK
    workspace / thread-pool start-up)."""
    best, out = float("inf"), None
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn(*a)
        best = min(best, time.perf_counter() - t0)
    return best, out


def warm(nb: int) -> None:
    """Spin up the BLAS / LAPACK thread pool and workspaces once."""
    a = np.random.default_rng(0).standard_normal((nb, nb))
    sla.svd(a, full_matrices=False, check_finite=False, lapack_driver="gesdd")
    np.linalg.qr(a)
    a @ a


def estimate_eval_seconds(xy, z, theta, nb, acc, pair_budget: int = 14) -> tuple[float, str]:
    n = xy.shape[0]
    nb = min(nb, n)
    if not acc:
        t0 = time.perf_counter()
        orc.log_likelihood(xy, z, theta, nb, None)
        return time.perf_counter() - t0, "full dense evaluation (assembly + Cholesky + solve)"
    b = orc.tile_bounds(n, nb)
    t = len(b)
    mid = t // 2
    warm(nb)

    def tile(i, j):
        return orc.matern_block(xy[b[i][0]:b[i][1]], xy[b[j][0]:b[j][1]], theta)

    # generation + compression per offset; keep tiles of column 0 and the
    # compressed tiles for recompression samples
    comp = {}
    gen_total = 0.0
    rank_by_off = {}
    for d in range(1, t):
        i, j = min(t - 1, mid + d // 2 + (d % 2)), None
        j = i - d
        if j < 0:
            i, j = d, 0
        dt, lr = _t(lambda a: orc.compress_tile(a, acc), tile(i, j))
        gen_total += dt * (t - d)
        comp[d] = lr
        rank_by_off[d] = lr[0].shape[1]
    # diagonal tile POTRF
    d0 = tile(mid, mid)
    dt_p, lkk = _t(orc.potrf_tile, d0, mid)
    potrf_total = dt_p * t
    # TRSM + SYRK on a representative panel tile (offset 1)
    u, v = comp[1]
    dt_trsm, v2 = _t(lambda: sla.solve_triangular(lkk, v, lower=True, check_finite=False))
    dt_syrk, _ = _t(lambda: (u @ (v2.T @ v2)) @ u.T)
    panel_total = (dt_trsm + dt_syrk) * t * (t - 1) / 2
    # recompressions: offsets (d1, d2) on a spread grid
    ds = sorted({1, 2, 3, 4, 6, 9, 13, t - 2} & set(range(1, t - 1)))
    pairs = [(d1, d2) for d1 in ds for d2 in ds if d1 + d2 <= t - 1]
    if len(pairs) > pair_budget:
        idx = np.linspace(0, len(pairs) - 1, pair_budget).round().astype(int)
        pairs = [pairs[k] for k in sorted(set(idx))]
    samples = []
    for d1, d2 in pairs:
        u0, v0 = comp[d1]                 # tile (i, j)
        ui, vi = comp[d1 + d2]            # tile (i, k)
        uj, vj = comp[d2]                 # tile (j, k)
        if ui.shape[1] == 0 or uj.shape[1] == 0:
            continue
        m0, m1 = u0.shape[0], vj.shape[0]
        vi = vi[:m1] if vi.shape[0] >= m1 else np.vstack([vi, np.zeros((m1 - vi.shape[0], vi.shape[1]))])
        ui = ui[:m0] if ui.shape[0] >= m0 else np.vstack([ui, np.zeros((m0 - ui.shape[0], ui.shape[1]))])
        dt, _ = _t(lambda: orc.recompress(u0, v0, -(ui @ (vi.T @ vj)), uj, acc))
        samples.append((u0.shape[1] + uj.shape[1], dt))
    samples.sort()
    ks = np.array([s[0] for s in samples], float)
    ts = np.array([s[1] for s in samples], float)
    upd_total = 0.0
    for d1 in range(1, t):
        for d2 in range(1, t - d1):
            cnt = t - d1 - d2
            K = rank_by_off[d1] + rank_by_off[d2]
            upd_total += cnt * float(np.interp(K, ks, ts))
    solve_est = 2e-9 * n * n / 8  # forward solve: a few GB/s over the stored factor (upper bound)
    total = gen_total + potrf_total + panel_total + upd_total + solve_est
    desc = (f"stratified sample: {t - 1} tile compressions (one per offset), 1 POTRF, 1 TRSM+SYRK, "
            f"{len(samples)} recompressions over (d1,d2) offset pairs, extrapolated to "
            f"{t * (t - 1) // 2} tiles and {t * (t - 1) * (t - 2) // 6} updates")
    return total, desc


def calibration() -> dict:
    """The estimator against full timed runs of the unmodified reference: the
    C3 TLR(1e-7) golden run (tests/golden/c3_tlr.json, one evaluation on the
    build container's host cores) and the estimator on the same host
    (profiles/r02_reference_calibration.json)."""
    from pathlib import Path
    import json
    root = Path(__file__).resolve().parents[1]
    out = {}
    g = root / "tests" / "golden" / "c3_tlr.json"
    if g.exists():
        d = json.loads(g.read_text())["C3"]
        out["full_reference_c3_tlr_s"] = d.get("seconds")
        out["full_reference_host"] = d.get("host", "build container, 8 cores")
    c = root / "profiles" / "r02_reference_calibration.json"
    if c.exists():
        out.update(json.loads(c.read_text()))
    return out


def host_threads() -> int:
    return int(os.environ.get("OPENBLAS_NUM_THREADS") or os.cpu_count() or 1)
