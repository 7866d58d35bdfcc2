"""CPU oracle for the TLR Gaussian log-likelihood hot path.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this module,
and only as the checker or the timed CPU reference arm.  The product path
(`paper_1804_09137_b200`) never imports it and has no CPU fallback.

This is a numpy/scipy restatement of the reference package `tlrgeo`
(/root/reference/pkg/src/tlrgeo, pure Python + numba + LAPACK).  Each
function cites the reference file:line it restates.  It is *pinned* against
fixtures produced by the unmodified reference (`tests/golden/make_goldens.py`,
run in the build container where /root/reference exists) by
`tests/test_oracle.py`: K_nu values, locations, covariance tiles, compression
ranks, and log-likelihood / solve / kriging values.

Arithmetic notes (parity-relevant):
  * K_nu is evaluated exactly (Temme series for x<=2, Thompson-Barnett CF2
    for x>2, forward recurrence), vectorised over all entries of a tile; the
    reference uses a cubic-spline profile of the same function for n>=256
    (tilestore.py:166-178) whose per-entry error is <=1e-12 and whose effect
    on the log-likelihood is <=2.3e-13 relative.
  * LAPACK drivers match the reference's: gesdd for SVDs, geqrf/orgqr through
    numpy.linalg.qr, potrf, trsm via scipy.linalg.solve_triangular.
"""
from __future__ import annotations

import math

import numpy as np
import scipy.linalg as sla

LOG_2PI = math.log(2.0 * math.pi)          # stats.py:28
KERNEL_CUTOFF_T = 700.0                     # kernels.py:31
_EPS_SERIES = 1e-15                         # kernels.py:78
_MAX_ITER = 1000                            # kernels.py:79
# Taylor coefficients of gam1(mu) near 0 (kernels.py:74-76)
_G1 = (-0.5772156649015328606, 0.0420026350340952355, 0.0421977345555443367)


class NotPositiveDefiniteError(Exception):
    """linalg.py:20-33 — failed pivot; carries (tile_index, pivot_index)."""

    def __init__(self, tile_index: int, pivot_index: int):
        self.tile_index = tile_index
        self.pivot_index = pivot_index
        super().__init__(f"covariance not positive definite at tile {tile_index}, "
                         f"pivot {pivot_index}; consider adding a nugget")


# --------------------------------------------------------------------------
# geometry (geometry.py:186-206)
# --------------------------------------------------------------------------
def generate_locations(n: int, seed: int) -> np.ndarray:
    """Jittered ceil(sqrt n) grid, row-major; (n,2) float64.  geometry.py:186-206."""
    g = math.isqrt(n)
    g += g * g < n
    jitter = np.random.default_rng(seed).uniform(-0.4, 0.4, (n, 2))
    k = np.arange(n)
    x = (k // g + 1 - 0.5 + jitter[:, 0]) / g
    y = (k % g + 1 - 0.5 + jitter[:, 1]) / g
    return np.column_stack((x, y))


# --------------------------------------------------------------------------
# modified Bessel K_nu, vectorised restatement of kernels.py:82-174
# --------------------------------------------------------------------------
def _temme_constants(mu: float):
    """kernels.py:82-93."""
    gp = 1.0 / math.gamma(1.0 + mu)
    gm = 1.0 / math.gamma(1.0 - mu)
    if abs(mu) < 1e-2:
        m2 = mu * mu
        g1 = _G1[0] + m2 * (_G1[1] + m2 * _G1[2])
    else:
        g1 = (gm - gp) / (2.0 * mu)
    return gp, gm, g1, 0.5 * (gm + gp)


def _series_pair(mu, x, consts):
    """Temme series, x<=2: (K_mu, K_mu+1).  kernels.py:96-123 (vectorised; an
    element stops updating on the iteration the scalar loop would break)."""
    gp, gm, g1, g2 = consts
    half = 0.5 * x
    pm = math.pi * mu
    fact = 1.0 if abs(pm) < 1e-15 else pm / math.sin(pm)
    d = -np.log(half)
    e = mu * d
    with np.errstate(invalid="ignore", divide="ignore"):
        f2 = np.where(np.abs(e) < 1e-15, 1.0, np.sinh(e) / e)
    ff = fact * (g1 * np.cosh(e) + g2 * f2 * d)
    ks = ff.copy()
    ee = np.exp(e)
    p = 0.5 * ee / gp
    q = 0.5 / (ee * gm)
    c = np.ones_like(x)
    d2 = half * half
    ks1 = p.copy()
    live = np.ones(x.shape, bool)
    for i in range(1, _MAX_ITER):
        if not live.any():
            break
        ff = np.where(live, (i * ff + p + q) / (i * i - mu * mu), ff)
        c = np.where(live, c * d2 / i, c)
        p = np.where(live, p / (i - mu), p)
        q = np.where(live, q / (i + mu), q)
        dk = c * ff
        ks = np.where(live, ks + dk, ks)
        ks1 = np.where(live, ks1 + c * (p - i * ff), ks1)
        live &= ~(np.abs(dk) < np.abs(ks) * _EPS_SERIES)
    return ks, ks1 * (2.0 / x)


def _cf2_pair(mu, x):
    """Thompson-Barnett continued fraction, x>2.  kernels.py:126-157."""
    b = 2.0 * (1.0 + x)
    d = 1.0 / b
    h = d.copy()
    dh = d.copy()
    q1 = np.zeros_like(x)
    q2 = np.ones_like(x)
    a1 = 0.25 - mu * mu
    q = np.full_like(x, a1)
    c = np.full_like(x, a1)
    a = np.full_like(x, -a1)
    s = 1.0 + q * dh
    live = np.ones(x.shape, bool)
    for i in range(2, _MAX_ITER):
        if not live.any():
            break
        a_n = a - 2.0 * (i - 1)
        c_n = -a_n * c / i
        qn = (q1 - b * q2) / a_n
        q_n = q + c_n * qn
        b_n = b + 2.0
        d_n = 1.0 / (b_n + a_n * d)
        dh_n = (b_n * d_n - 1.0) * dh
        h_n = h + dh_n
        ds = q_n * dh_n
        s_n = s + ds
        a = np.where(live, a_n, a); c = np.where(live, c_n, c)
        q1, q2 = np.where(live, q2, q1), np.where(live, qn, q2)
        q = np.where(live, q_n, q); b = np.where(live, b_n, b)
        d = np.where(live, d_n, d); dh = np.where(live, dh_n, dh)
        h = np.where(live, h_n, h); s = np.where(live, s_n, s)
        live &= ~(np.abs(ds / s) < _EPS_SERIES)
    h = a1 * h
    k0 = np.sqrt(math.pi / (2.0 * x)) * np.exp(-x) / s
    return k0, k0 * (mu + x + 0.5 - h) / x


def bessel_k(nu: float, x) -> np.ndarray:
    """K_nu(x), nu in (0,5], x>0.  kernels.py:160-174 (`_kv_raw`)."""
    x = np.atleast_1d(np.asarray(x, dtype=float))
    nl = int(nu + 0.5)
    mu = nu - nl
    k0 = np.empty_like(x)
    k1 = np.empty_like(x)
    lo = x <= 2.0
    if lo.any():
        k0[lo], k1[lo] = _series_pair(mu, x[lo], _temme_constants(mu))
    if (~lo).any():
        k0[~lo], k1[~lo] = _cf2_pair(mu, x[~lo])
    for i in range(nl):
        k0, k1 = k1, (mu + i + 1.0) * (2.0 / x) * k1 + k0
    return k0


def matern_prefactor(theta1: float, nu: float) -> float:
    """kernels.py:59-62."""
    return theta1 / (2.0 ** (nu - 1.0) * math.gamma(nu))


def matern_t(t, theta1: float, nu: float) -> np.ndarray:
    """Kernel of the scaled distance t = r/theta2.  kernels.py:177-188."""
    t = np.asarray(t, dtype=float)
    out = np.full(t.shape, theta1)
    mid = (t > 0.0) & (t <= KERNEL_CUTOFF_T)
    out[t > KERNEL_CUTOFF_T] = 0.0
    if mid.any():
        tm = t[mid]
        with np.errstate(over="ignore", invalid="ignore"):
            v = matern_prefactor(theta1, nu) * tm ** nu * bessel_k(nu, tm)
        bad = ~np.isfinite(v) | (v > theta1)
        v[bad] = theta1
        out[mid] = v
    return out


def distance_block(rows_xy: np.ndarray, cols_xy: np.ndarray, radius: float = 0.0) -> np.ndarray:
    """Pairwise distances.  radius == 0: Euclidean (kernels.py:436-443);
    radius > 0: haversine on (lon, lat) degrees through the KernelView
    (lat, lon radians, cos lat; geometry.py:106-122) in the operation order
    of kernels.py:461-473."""
    if radius == 0.0:
        dx = rows_xy[:, 0:1] - cols_xy[None, :, 0]
        dy = rows_xy[:, 1:2] - cols_xy[None, :, 1]
        return np.sqrt(dx * dx + dy * dy)
    plat, plon = np.radians(rows_xy[:, 1])[:, None], np.radians(rows_xy[:, 0])[:, None]
    qlat, qlon = np.radians(cols_xy[:, 1])[None, :], np.radians(cols_xy[:, 0])[None, :]
    sp = np.sin(0.5 * (qlat - plat))
    sl = np.sin(0.5 * (qlon - plon))
    a = np.minimum(sp * sp + np.cos(plat) * np.cos(qlat) * sl * sl, 1.0)
    return (2.0 * radius) * np.arcsin(np.sqrt(a))


def matern_block(rows_xy: np.ndarray, cols_xy: np.ndarray, theta, radius: float = 0.0) -> np.ndarray:
    """Dense kernel block, no nugget.  kernels.py:436-491 / 494-530."""
    th1, th2, nu = theta[0], theta[1], theta[2]
    t = distance_block(rows_xy, cols_xy, radius) * (1.0 / th2)
    return matern_t(t, th1, nu)


# --------------------------------------------------------------------------
# tile grid + assembly (tilestore.py:25-59, 181-223)
# --------------------------------------------------------------------------
def tile_bounds(n: int, nb: int):
    """TileGrid.bounds for every tile.  tilestore.py:36-44."""
    t = -(-n // nb)
    return [(i * nb, min((i + 1) * nb, n)) for i in range(t)]


def truncation_rank(s: np.ndarray, eps: float) -> int:
    """Smallest k with ||s[k:]|| <= eps ||s||, tail summed from the small end.
    compression.py:26-36."""
    if s.size == 0:
        return 0
    sq = s * s
    total = float(sq.sum())
    if total == 0.0:
        return 0
    tail = np.cumsum(sq[::-1])[::-1]
    hit = np.flatnonzero(tail <= eps * eps * total)
    return int(hit[0]) if hit.size else int(s.size)


def compress_tile(a: np.ndarray, eps: float):
    """gesdd + truncation; returns (u*s, v).  compression.py:39-51."""
    u, s, vt = sla.svd(a, full_matrices=False, check_finite=False, lapack_driver="gesdd")
    k = truncation_rank(s, eps)
    return u[:, :k] * s[:k], vt[:k].T.copy()


def recompress(u1, v1, u2, v2, eps: float):
    """QR of stacked factors + core SVD + noise floor.  compression.py:54-81."""
    if u1.shape[1] + u2.shape[1] == 0:
        return u1, v1
    qu, ru = np.linalg.qr(np.hstack((u1, u2)))
    qv, rv = np.linalg.qr(np.hstack((v1, v2)))
    w, s, zt = sla.svd(ru @ rv.T, full_matrices=False, check_finite=False,
                       lapack_driver="gesdd")
    floor = 50 * np.finfo(float).eps * np.linalg.norm(ru) * np.linalg.norm(rv)
    s = s[s > floor]
    k = truncation_rank(s, eps)
    return qu @ (w[:, :k] * s[:k]), qv @ zt[:k].T


def assemble(xy: np.ndarray, theta, nb: int, acc: float | None, radius: float = 0.0):
    """Lower-triangle tile assembly; TLR mode compresses each off-diagonal tile.
    tilestore.py:181-223.  Returns (diag list, lower dict)."""
    n = xy.shape[0]
    bnds = tile_bounds(n, nb)
    nugget = theta[3] if len(theta) > 3 else 0.0
    diag, lower = [], {}
    for i, (r0, r1) in enumerate(bnds):
        d = matern_block(xy[r0:r1], xy[r0:r1], theta, radius)
        if nugget:
            d[np.diag_indices_from(d)] += nugget
        diag.append(d)
        for j in range(i):
            c0, c1 = bnds[j]
            blk = matern_block(xy[r0:r1], xy[c0:c1], theta, radius)
            lower[(i, j)] = compress_tile(blk, acc) if acc else blk
    return diag, lower


# --------------------------------------------------------------------------
# tile Cholesky (linalg.py:36-140)
# --------------------------------------------------------------------------
def potrf_tile(a: np.ndarray, tile_index: int) -> np.ndarray:
    """LAPACK dpotrf lower; info -> NotPositiveDefiniteError.  linalg.py:36-45."""
    (potrf,) = sla.get_lapack_funcs(("potrf",), (a,))
    c, info = potrf(a, lower=1, overwrite_a=0)
    if info != 0:
        raise NotPositiveDefiniteError(tile_index, int(info) - 1)
    return np.tril(c)


def cholesky(diag, lower, acc: float | None):
    """Right-looking tile Cholesky, dense (linalg.py:82-103) or TLR with eager
    per-(i,j) recompression in k order (linalg.py:106-140).
    Returns (diag_factors, lower_factors, log_det)."""
    t = len(diag)
    D = [d.copy() for d in diag]
    L = {k: (v if acc else v.copy()) for k, v in lower.items()}
    log_det = 0.0
    for k in range(t):
        lkk = potrf_tile(D[k], k)
        D[k] = lkk
        log_det += 2.0 * float(np.sum(np.log(np.diag(lkk))))
        if not acc:
            for i in range(k + 1, t):
                L[(i, k)] = sla.solve_triangular(lkk, L[(i, k)].T, lower=True,
                                                 check_finite=False).T
            for j in range(k + 1, t):
                ljk = L[(j, k)]
                D[j] -= ljk @ ljk.T
                for i in range(j + 1, t):
                    L[(i, j)] -= L[(i, k)] @ ljk.T
            continue
        for i in range(k + 1, t):
            u, v = L[(i, k)]
            if u.shape[1]:
                L[(i, k)] = (u, sla.solve_triangular(lkk, v, lower=True, check_finite=False))
        for j in range(k + 1, t):
            uj, vj = L[(j, k)]
            if uj.shape[1]:
                D[j] -= (uj @ (vj.T @ vj)) @ uj.T
            for i in range(j + 1, t):
                ui, vi = L[(i, k)]
                if ui.shape[1] == 0 or uj.shape[1] == 0:
                    continue
                u0, v0 = L[(i, j)]
                L[(i, j)] = recompress(u0, v0, -(ui @ (vi.T @ vj)), uj, acc)
    return D, L, log_det


def _apply(tile, x, transpose=False):
    if isinstance(tile, tuple):
        u, v = tile
        if u.shape[1] == 0:
            return 0.0
        return v @ (u.T @ x) if transpose else u @ (v.T @ x)
    return tile.T @ x if transpose else tile @ x


def forward_solve(D, L, n, nb, rhs):
    """L y = rhs by tile rows.  linalg.py:166-177."""
    y = np.array(rhs, dtype=float, copy=True)
    b = tile_bounds(n, nb)
    for i, (r0, r1) in enumerate(b):
        acc = y[r0:r1]
        for j in range(i):
            acc = acc - _apply(L[(i, j)], y[b[j][0]:b[j][1]])
        y[r0:r1] = sla.solve_triangular(D[i], acc, lower=True, check_finite=False)
    return y


def backward_solve(D, L, n, nb, rhs):
    """L^T x = rhs, reverse tile order.  linalg.py:180-192."""
    x = np.array(rhs, dtype=float, copy=True)
    b = tile_bounds(n, nb)
    t = len(b)
    for i in range(t - 1, -1, -1):
        r0, r1 = b[i]
        acc = x[r0:r1]
        for j in range(i + 1, t):
            acc = acc - _apply(L[(j, i)], x[b[j][0]:b[j][1]], transpose=True)
        x[r0:r1] = sla.solve_triangular(D[i], acc, lower=True, trans="T",
                                        check_finite=False)
    return x


def log_likelihood(xy, z, theta, nb, acc=None, radius=0.0):
    """-0.5 (n log 2pi + log|Sigma| + z' Sigma^-1 z).  stats.py:96-112.
    Returns (ll, log_det, quad)."""
    n = xy.shape[0]
    nb = min(nb, n)
    D, L, log_det = cholesky(*assemble(xy, theta, nb, acc, radius), acc)
    y = forward_solve(D, L, n, nb, z)
    quad = float(y @ y)
    return -0.5 * (n * LOG_2PI + log_det + quad), log_det, quad


def sample_measurements(xy, theta, seed: int, radius: float = 0.0) -> np.ndarray:
    """z = L w, dense nb=min(200,n), w ~ N(0,1) from default_rng(seed).
    stats.py:115-133."""
    n = xy.shape[0]
    nb = min(200, n)
    D, L, _ = cholesky(*assemble(xy, theta, nb, None, radius), None)
    w = np.random.default_rng(seed).standard_normal(n)
    b = tile_bounds(n, nb)
    out = np.zeros(n)
    for i, (r0, r1) in enumerate(b):
        out[r0:r1] = D[i] @ w[r0:r1]
        for j in range(i):
            out[r0:r1] += L[(i, j)] @ w[b[j][0]:b[j][1]]
    return out


def predict(known_xy, z, unknown_xy, theta, nb, acc=None, radius=0.0):
    """Kriging mean S12 S22^-1 z.  predict.py:65-87 (mean branch)."""
    n = known_xy.shape[0]
    nb = min(nb, n)
    D, L, _ = cholesky(*assemble(known_xy, theta, nb, acc, radius), acc)
    w = backward_solve(D, L, n, nb, forward_solve(D, L, n, nb, z))
    return matern_block(unknown_xy, known_xy, theta, radius) @ w


# --------------------------------------------------------------------------
# bounded Nelder-Mead MLE (stats.py:144-251) — checker for the device driver
# --------------------------------------------------------------------------
def mle_fit(objective, bounds, theta0=None, max_iterations=100, tol=1e-9):
    """Returns (best theta, best loglik, iterations, converged, trace of thetas)."""
    lo = [b[0] for b in bounds]
    hi = [b[1] for b in bounds]
    clamp = lambda x: np.array([min(max(x[d], lo[d]), hi[d]) for d in range(len(x))])
    thetas = []

    def neg(x):
        thetas.append(tuple(float(v) for v in x))
        ll = objective(x)
        return -ll if math.isfinite(ll) else math.inf

    x0 = clamp(np.asarray(theta0 if theta0 is not None else [math.sqrt(a * b) for a, b in bounds],
                          dtype=float))
    verts = [x0.copy()]
    for d in range(x0.size):                              # stats.py:148-158
        step = 0.25 * x0[d]
        v = x0.copy()
        if v[d] + step > hi[d]:
            step = -step
        v[d] = min(max(v[d] + step, lo[d]), hi[d])
        verts.append(v)
    fv = [neg(v) for v in verts]
    it, conv = 0, False
    while it < max_iterations:                            # stats.py:206-237
        o = np.argsort(fv, kind="stable")
        verts = [verts[k] for k in o]
        fv = [fv[k] for k in o]
        a, b = fv[0], fv[-1]
        spread = (2.0 * abs(b - a) / (abs(b) + abs(a) + 1e-300)
                  if math.isfinite(a) and math.isfinite(b) else math.inf)
        if spread <= tol:
            conv = True
            break
        it += 1
        c = np.mean(verts[:-1], axis=0)
        xr = clamp(c + (c - verts[-1]))
        fr = neg(xr)
        if fv[0] <= fr < fv[-2]:
            verts[-1], fv[-1] = xr, fr
        elif fr < fv[0]:
            xe = clamp(c + 2.0 * (xr - c))
            fe = neg(xe)
            verts[-1], fv[-1] = (xe, fe) if fe < fr else (xr, fr)
        else:
            xc = clamp(c + 0.5 * ((xr if fr < fv[-1] else verts[-1]) - c))
            fc = neg(xc)
            if fc < min(fr, fv[-1]):
                verts[-1], fv[-1] = xc, fc
            else:
                for k in range(1, len(verts)):
                    verts[k] = clamp(verts[0] + 0.5 * (verts[k] - verts[0]))
                    fv[k] = neg(verts[k])
    best = int(np.argmin(fv))
    return verts[best], -fv[best], it, conv, thetas
