"""Drop-in Python surface for the reference's likelihood / kriging path.

Mirrors (names, argument meaning, error behaviour) the reference package
`tlrgeo` (/root/reference/pkg/src/tlrgeo):

  MaternParams          kernels.py:34-65
  Euclidean, GreatCircle geometry.py:16-33
  LocationSet           geometry.py:78-149 (both metrics)
  generate_locations    geometry.py:186-206
  LikelihoodConfig      stats.py:41-70   (+ max_rank, ngpus)
  log_likelihood        stats.py:103-112
  PredictionProblem     predict.py:20-48
  predict (mean)        predict.py:65-87
  NotPositiveDefiniteError linalg.py:20-33
  bessel_k, matern_block, compress_tile (component entry points)

Every numerical call goes through libtlrb200.so (hand-written sm_100a CUDA);
nothing here computes on the CPU beyond argument marshalling.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import TlrbStats, dptr, iptr

THETA3_MAX = 5.0
DEFAULT_NB_DENSE = 200          # tilestore.py:19
DEFAULT_NB_TLR = 400            # tilestore.py:20
LOG_2PI = math.log(2.0 * math.pi)


class NotPositiveDefiniteError(Exception):
    """Same contract as the reference (linalg.py:20-33)."""

    def __init__(self, tile_index: int, pivot_index: int):
        self.tile_index = tile_index
        self.pivot_index = pivot_index
        super().__init__(
            f"covariance not positive definite at tile {tile_index}, "
            f"pivot {pivot_index}; consider adding a nugget")


class DeviceError(RuntimeError):
    """CUDA / out-of-memory failure inside libtlrb200.so."""


@dataclass(frozen=True)
class MaternParams:
    """(variance, range, smoothness) + nugget; validation of kernels.py:43-57."""

    theta1: float
    theta2: float
    theta3: float
    nugget: float = 0.0

    def __post_init__(self):
        vals = (self.theta1, self.theta2, self.theta3, self.nugget)
        if not all(math.isfinite(v) for v in vals):
            raise ValueError(f"non-finite Matern parameters: {vals}")
        if self.theta1 <= 0 or self.theta2 <= 0 or self.theta3 <= 0:
            raise ValueError(f"theta components must be strictly positive, got "
                             f"({self.theta1}, {self.theta2}, {self.theta3})")
        if self.theta3 > THETA3_MAX:
            raise ValueError(f"smoothness theta3={self.theta3} exceeds supported bound {THETA3_MAX}")
        if self.nugget < 0:
            raise ValueError(f"nugget must be non-negative, got {self.nugget}")

    @property
    def prefactor(self) -> float:
        return self.theta1 / (2.0 ** (self.theta3 - 1.0) * math.gamma(self.theta3))

    def as_tuple(self):
        return (self.theta1, self.theta2, self.theta3, self.nugget)


EARTH_RADIUS_KM = 6371.0       # geometry.py:16


@dataclass(frozen=True)
class Euclidean:
    """Planar distance (geometry.py:19-21)."""


@dataclass(frozen=True)
class GreatCircle:
    """Haversine distance on a sphere of `radius`; coordinates are
    (lon, lat) in degrees (geometry.py:24-31)."""

    radius: float = EARTH_RADIUS_KM

    def __post_init__(self):
        if not (self.radius > 0) or not math.isfinite(self.radius):
            raise ValueError(f"sphere radius must be positive, got {self.radius}")


def sphere_radius(metric) -> float:
    """0.0 for Euclidean, the sphere radius for great circle.  Accepts this
    module's metrics and the reference's (matched by class name)."""
    name = type(metric).__name__
    if metric is None or name == "Euclidean":
        return 0.0
    if name == "GreatCircle":
        return float(metric.radius)
    raise ValueError(f"unsupported metric {metric!r}")


class LocationSet:
    """Ordered set of distinct locations, (n, 2), with a metric
    (geometry.py:78-97: same validation and errors)."""

    def __init__(self, coords, metric=None):
        metric = Euclidean() if metric is None else metric
        coords = np.ascontiguousarray(coords, dtype=float)
        if coords.ndim != 2 or coords.shape[1] != 2 or coords.shape[0] == 0:
            raise ValueError(f"coords must be a non-empty (n, 2) array, got {coords.shape}")
        if not np.isfinite(coords).all():
            raise ValueError("locations must be finite")
        if sphere_radius(metric) > 0:
            lon, lat = coords[:, 0], coords[:, 1]
            if (np.abs(lon) > 180).any() or (np.abs(lat) > 90).any():
                raise ValueError("great-circle coordinates must satisfy "
                                 "lon in [-180, 180], lat in [-90, 90]")
        if np.unique(coords, axis=0).shape[0] != coords.shape[0]:
            raise ValueError("locations must be pairwise distinct")
        coords.setflags(write=False)
        self.coords = coords
        self.metric = metric

    def __len__(self) -> int:
        return self.coords.shape[0]


def generate_locations(n: int, seed: int) -> LocationSet:
    """Jittered ceil(sqrt n) grid in [0,1]^2, row-major (geometry.py:186-206)."""
    if n < 1:
        raise ValueError(f"n must be >= 1, got {n}")
    g = math.isqrt(n)
    if g * g < n:
        g += 1
    off = np.random.default_rng(seed).uniform(-0.4, 0.4, (n, 2))
    idx = np.arange(n)
    coords = np.column_stack(((idx // g + 0.5 + off[:, 0]) / g,
                              (idx % g + 0.5 + off[:, 1]) / g))
    return LocationSet(coords)


@dataclass(frozen=True)
class LikelihoodConfig:
    """stats.py:41-70 fields used by the likelihood, plus the build's
    `max_rank` (tile storage cap; <=0/None = uncapped) and `ngpus`."""

    mode: str = "dense"
    accuracy: float | None = None
    nb: int | None = None
    nugget: float = 0.0
    bounds: tuple = ((0.01, 5.0), (0.001, 3.0), (0.1, 3.0))
    theta0: tuple | None = None
    max_iterations: int = 100
    tol: float = 1e-9
    profile: object = "auto"
    max_rank: int | None = None
    ngpus: int = 1

    def __post_init__(self):
        if self.mode not in ("dense", "tlr"):
            raise ValueError(f"unknown mode {self.mode!r}")
        if self.mode == "tlr" and self.accuracy is None:
            raise ValueError("tlr mode requires an accuracy threshold")
        if self.mode == "tlr" and not (0.0 < self.accuracy < 1.0):
            raise ValueError(f"accuracy must lie in (0, 1), got {self.accuracy}")
        for lo, hi in self.bounds:   # stats.py:60-62
            if not (0.0 < lo < hi):
                raise ValueError(f"invalid bounds ({lo}, {hi})")
        if self.ngpus < 1:
            raise ValueError(f"ngpus must be >= 1, got {self.ngpus}")

    def tile_size(self) -> int:
        if self.nb is not None:
            return self.nb
        return DEFAULT_NB_DENSE if self.mode == "dense" else DEFAULT_NB_TLR

    def label(self) -> str:
        """Canonical mode label (stats.py:68-69, 266-270): "dense" or e.g. "tlr:1e-5"."""
        if self.mode == "dense":
            return "dense"
        return "tlr:" + f"{self.accuracy:g}".replace("e-0", "e-").replace("e+0", "e+")


# --------------------------------------------------------------------------
class Handle:
    """Owns one libtlrb200 handle: locations resident on the device, tile
    arenas reused across evaluations (one MLE run = one handle)."""

    def __init__(self, coords: np.ndarray, nb: int, max_rank: int = 0, ngpus: int = 1,
                 device: int = 0, dist: tuple | None = None, radius: float = 0.0,
                 group: tuple | None = None):
        """dist = (rank, world, P, Q, nccl_id_bytes): 2D block-cyclic multi-GPU
        handle (one process per GPU); see `distributed_handle`.  ngpus > 1:
        one handle driving devices device .. device + ngpus - 1 from this
        process.  group = (devices, P, Q, backend): the same schedule with
        len(devices) ranks in this process (devices may repeat; backend
        _lib.TLRB_BACKEND_LOOPBACK runs several ranks on one GPU), see
        `group_handle`.  radius > 0: great-circle metric on that sphere,
        coords = (lon, lat) degrees."""
        self.lib = _lib.load()
        xy = np.ascontiguousarray(coords, dtype=np.float64)
        self.n = xy.shape[0]
        self.nb = int(min(nb, self.n))
        err = np.zeros(1, np.int32)
        if group is not None:
            devs, P, Q, backend = group
            d = np.ascontiguousarray(devs, dtype=np.int32)
            self.h = self.lib.tlrb_create_group(dptr(xy), self.n, self.nb, int(max_rank or 0), iptr(d),
                                                int(d.size), int(P), int(Q), int(backend), iptr(err))
        elif dist is None:
            self.h = self.lib.tlrb_create(dptr(xy), self.n, self.nb, int(ngpus), int(max_rank or 0),
                                          int(device), iptr(err))
        else:
            rank, world, P, Q, nid = dist
            self.h = self.lib.tlrb_create_dist(dptr(xy), self.n, self.nb, int(max_rank or 0), int(device),
                                               int(rank), int(world), int(P), int(Q), bytes(nid), iptr(err))
        if not self.h:
            raise (ValueError if err[0] == _lib.TLRB_ERR_ARG else DeviceError)(
                f"tlrb_create failed (code {int(err[0])})")
        self.last_stats: dict | None = None
        self.radius = float(radius)
        if self.radius:
            rc = self.lib.tlrb_set_metric(self.h, self.radius)
            if rc:
                self._raise(rc)

    def close(self):
        if getattr(self, "h", None):
            self.lib.tlrb_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _raise(self, rc: int):
        tile = np.zeros(1, np.int32)
        piv = np.zeros(1, np.int32)
        buf = C.create_string_buffer(512)
        self.lib.tlrb_last_error(self.h, iptr(tile), iptr(piv), buf, 512)
        if rc == _lib.TLRB_ERR_NPD:
            raise NotPositiveDefiniteError(int(tile[0]), int(piv[0]))
        if rc == _lib.TLRB_ERR_ARG:
            raise ValueError(buf.value.decode() or "invalid argument")
        raise DeviceError(buf.value.decode() or f"libtlrb200 error {rc}")

    def loglik(self, z: np.ndarray, p: MaternParams, acc: float | None):
        z = np.ascontiguousarray(z, dtype=np.float64)
        out = np.zeros(3)
        st = TlrbStats()
        rc = self.lib.tlrb_loglik(self.h, dptr(z), p.theta1, p.theta2, p.theta3, p.nugget,
                                  float(acc or 0.0), dptr(out[0:]), dptr(out[1:]), dptr(out[2:]),
                                  C.byref(st))
        if rc:
            self._raise(rc)
        self.last_stats = st.as_dict()
        return float(out[0]), float(out[1]), float(out[2])

    def loglik_device(self, z_ptr: int, p: MaternParams, acc: float | None):
        out = np.zeros(3)
        st = TlrbStats()
        rc = self.lib.tlrb_loglik_device(self.h, C.c_void_p(z_ptr), p.theta1, p.theta2, p.theta3,
                                         p.nugget, float(acc or 0.0), dptr(out[0:]), dptr(out[1:]),
                                         dptr(out[2:]), C.byref(st))
        if rc:
            self._raise(rc)
        self.last_stats = st.as_dict()
        return float(out[0]), float(out[1]), float(out[2])

    def factorize(self, p: MaternParams, acc: float | None):
        rc = self.lib.tlrb_factorize(self.h, p.theta1, p.theta2, p.theta3, p.nugget, float(acc or 0.0))
        if rc:
            self._raise(rc)

    def apply_factor(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty_like(x)
        rc = self.lib.tlrb_apply_factor(self.h, dptr(x), dptr(y))
        if rc:
            self._raise(rc)
        return y

    def solve(self, rhs: np.ndarray) -> np.ndarray:
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        x = np.empty_like(rhs)
        rc = self.lib.tlrb_solve(self.h, dptr(rhs), dptr(x))
        if rc:
            self._raise(rc)
        return x

    def predict(self, z, unknown_xy, p: MaternParams, acc: float | None) -> np.ndarray:
        z = np.ascontiguousarray(z, dtype=np.float64)
        u = np.ascontiguousarray(unknown_xy, dtype=np.float64)
        out = np.empty(u.shape[0])
        rc = self.lib.tlrb_predict(self.h, dptr(z), dptr(u), u.shape[0], p.theta1, p.theta2,
                                   p.theta3, p.nugget, float(acc or 0.0), dptr(out))
        if rc:
            self._raise(rc)
        return out

    @property
    def world(self) -> int:
        """Ranks behind this handle (1 unless it is a group handle)."""
        return int(self.lib.tlrb_group_size(self.h))

    def member_stats(self, member: int) -> dict:
        """The last evaluation's statistics of one rank of a group handle."""
        st = TlrbStats()
        if self.lib.tlrb_member_stats(self.h, int(member), C.byref(st)):
            raise ValueError(f"no member {member}")
        return st.as_dict()

    def predict_var(self, z, unknown_xy, p: MaternParams, acc: float | None):
        """(mean, conditional covariance) of the unknown sites (tlrb_predict_var)."""
        z = np.ascontiguousarray(z, dtype=np.float64)
        u = np.ascontiguousarray(unknown_xy, dtype=np.float64)
        m = u.shape[0]
        out = np.empty(m)
        cov = np.empty((m, m))
        rc = self.lib.tlrb_predict_var(self.h, dptr(z), dptr(u), m, p.theta1, p.theta2, p.theta3, p.nugget,
                                       float(acc or 0.0), dptr(out), dptr(cov))
        if rc:
            self._raise(rc)
        return out, cov.T.copy()   # column-major on the device

    def rank_map(self) -> np.ndarray:
        t = np.zeros(1, np.int32)
        self.lib.tlrb_rank_map(self.h, None, 0, iptr(t))
        tt = int(t[0])
        r = np.zeros(tt * tt, np.int32)
        self.lib.tlrb_rank_map(self.h, iptr(r), tt * tt, iptr(t))
        return r.reshape(tt, tt)


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    rc = _lib.load().tlrb_nccl_unique_id(buf, 128)
    if rc:
        raise DeviceError("ncclGetUniqueId failed")
    return buf.raw


def distributed_handle(coords, nb: int, max_rank: int = 0, P: int | None = None,
                       Q: int | None = None, device: int | None = None, radius: float = 0.0) -> Handle:
    """Handle over all ranks of the default torch.distributed group (one
    process per GPU): 2D block-cyclic tiles on a P x Q grid.
    Single process without torch.distributed: world = 1."""
    from .dist import grid_shape
    try:
        import torch.distributed as tdist
        on = tdist.is_available() and tdist.is_initialized()
    except ImportError:
        on = False
    rank, world = (tdist.get_rank(), tdist.get_world_size()) if on else (0, 1)
    if P is None or Q is None:
        P, Q = grid_shape(world)
    nid = nccl_unique_id() if rank == 0 else bytes(128)
    if on and world > 1:
        obj = [nid]
        tdist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    if device is None:
        import os
        device = int(os.environ.get("LOCAL_RANK", "0"))
    return Handle(coords, nb, max_rank, device=device, dist=(rank, world, P, Q, nid), radius=radius)


def group_handle(coords, nb: int, world: int, max_rank: int = 0, devices=None, P: int | None = None,
                 Q: int | None = None, backend: int | None = None, radius: float = 0.0) -> Handle:
    """`world` ranks of the 2D block-cyclic schedule inside this process, one
    host thread each per call (tlrb_create_group).  devices defaults to
    [0] * world with the loopback backend: the multi-GPU path executed on one
    GPU (its collectives are host rendezvous + stream-ordered device copies,
    no kernel waits on another rank)."""
    from .dist import grid_shape
    if P is None or Q is None:
        P, Q = grid_shape(world)
    devices = [0] * world if devices is None else list(devices)
    if backend is None:
        backend = _lib.TLRB_BACKEND_AUTO
    return Handle(coords, nb, max_rank, group=(devices, P, Q, backend), radius=radius)


_HANDLES: dict = {}   # insertion-ordered: least recently used first
_MAX_HANDLES = 2      # each handle owns arenas sized from free HBM: keep few alive


def _local_device() -> int:
    """One process per GPU (torchrun): single-GPU handles go to LOCAL_RANK's device."""
    import os
    return int(os.environ.get("LOCAL_RANK", "0"))


def _handle_key(coords: np.ndarray, nb: int, max_rank, ngpus, radius: float = 0.0):
    return (coords.__array_interface__["data"][0], coords.shape[0], int(nb), int(max_rank or 0),
            int(ngpus or 1), float(radius))


def _handle_for(coords: np.ndarray, nb: int, max_rank, ngpus, radius: float = 0.0) -> Handle:
    """Cached handle for (coords, nb, max_rank, ngpus, metric): an MLE run
    reuses one handle.  A small LRU: evicted handles are closed at once, so
    their device arenas are released before the next handle sizes its own."""
    key = _handle_key(coords, nb, max_rank, ngpus, radius)
    h = _HANDLES.pop(key, None)
    if h is None or h[0] is not coords:
        if h is not None:
            h[1].close()
        while len(_HANDLES) >= _MAX_HANDLES:
            old = _HANDLES.pop(next(iter(_HANDLES)))
            old[1].close()
        if ngpus and ngpus > 1 and _torch_distributed_world() > 1:
            # one process per GPU under torch.distributed: NCCL ranks
            h = (coords, distributed_handle(coords, nb, max_rank or 0, radius=radius))
        else:
            # one process driving ngpus devices (one host thread per device)
            h = (coords, Handle(coords, nb, max_rank or 0, ngpus=int(ngpus or 1),
                                device=_local_device(), radius=radius))
    _HANDLES[key] = h
    return h[1]


def close_handles() -> None:
    """Release every cached device handle (their arenas go back to the GPU)."""
    while _HANDLES:
        _, h = _HANDLES.popitem()
        h[1].close()


def _torch_distributed_world() -> int:
    try:
        import torch.distributed as tdist
        if tdist.is_available() and tdist.is_initialized():
            return tdist.get_world_size()
    except ImportError:
        pass
    return 1


def _coords_of(locs) -> np.ndarray:
    coords = getattr(locs, "coords", None)
    if coords is None:
        raise TypeError("locs must be a LocationSet (with .coords)")
    return coords


def _radius_of(locs) -> float:
    return sphere_radius(getattr(locs, "metric", None))


def log_likelihood(locs, z, p: MaternParams, cfg: LikelihoodConfig = LikelihoodConfig()) -> float:
    """Gaussian log-likelihood of z under Sigma(p); one device factorization.

    Same signature / errors as tlrgeo.stats.log_likelihood (stats.py:103-112).
    """
    z = np.asarray(z, dtype=float)
    n = len(locs)
    if z.shape != (n,):
        raise ValueError(f"measurement vector shape {z.shape} does not match n={n}")
    coords = _coords_of(locs)
    nb = min(cfg.tile_size(), n)
    h = _handle_for(coords, nb, cfg.max_rank, cfg.ngpus, _radius_of(locs))
    acc = cfg.accuracy if cfg.mode == "tlr" else None
    ll, _, _ = h.loglik(z, p, acc)
    return ll


def log_likelihood_parts(locs, z, p: MaternParams, cfg: LikelihoodConfig = LikelihoodConfig()):
    """(ll, log_det, quad, stats) — diagnostic variant of log_likelihood."""
    z = np.asarray(z, dtype=float)
    coords = _coords_of(locs)
    nb = min(cfg.tile_size(), len(locs))
    h = _handle_for(coords, nb, cfg.max_rank, cfg.ngpus, _radius_of(locs))
    ll, ld, q = h.loglik(z, p, cfg.accuracy if cfg.mode == "tlr" else None)
    return ll, ld, q, h.last_stats


def sample_measurements(locs, p_true: MaternParams, seed: int, accuracy: float | None = None,
                        nb: int | None = None, max_rank: int | None = None, ngpus: int = 1) -> np.ndarray:
    """One zero-mean field realisation z = L w (stats.py:115-133), w the
    reference's own default_rng(seed) standard normals drawn on the host.

    Default (the reference's recipe): dense tile Cholesky with
    nb = min(200, n) on the device.  accuracy = eps (the C4 /
    C5 inputs, where a dense factor does not fit): z = L~ w with L~ the TLR
    factor at eps (nb default 400, max_rank as in LikelihoodConfig), i.e. a
    field whose covariance is within eps of Sigma(p_true)."""
    coords = _coords_of(locs)
    n = coords.shape[0]
    if accuracy is None:
        tile = min(DEFAULT_NB_DENSE if nb is None else nb, n)
    else:
        if not (0.0 < accuracy < 1.0):
            raise ValueError(f"accuracy must lie in (0, 1), got {accuracy}")
        tile = min(DEFAULT_NB_TLR if nb is None else nb, n)
    h = Handle(coords, tile, max_rank or 0, ngpus=ngpus, device=_local_device(), radius=_radius_of(locs))
    try:
        h.factorize(p_true, accuracy)
        w = np.random.default_rng(seed).standard_normal(n)
        return h.apply_factor(w)
    finally:
        h.close()


@dataclass(frozen=True)
class PredictionProblem:
    """predict.py:20-48."""

    known: object
    z: np.ndarray
    unknown: object
    theta: MaternParams
    mode: str = "dense"
    accuracy: float | None = None
    nb: int | None = None
    max_rank: int | None = None

    def __post_init__(self):
        mk, mu = getattr(self.known, "metric", None), getattr(self.unknown, "metric", None)
        if sphere_radius(mk) != sphere_radius(mu):
            raise ValueError("known and unknown sets use different metrics")
        z = np.asarray(self.z, dtype=float)
        if z.shape != (len(self.known),):
            raise ValueError(f"measurement shape {z.shape} does not match {len(self.known)} locations")
        if self.mode not in ("dense", "tlr"):
            raise ValueError(f"unknown mode {self.mode!r}")
        if self.mode == "tlr" and self.accuracy is None:
            raise ValueError("tlr mode requires an accuracy threshold")

    def tile_size(self) -> int:
        if self.nb is not None:
            return self.nb
        return DEFAULT_NB_DENSE if self.mode == "dense" else DEFAULT_NB_TLR


def predict(p: PredictionProblem, with_variance: bool = False):
    """Kriging mean Sigma_12 Sigma_22^-1 z (predict.py:65-87); with_variance
    (dense mode only, like the reference) also returns the conditional
    covariance Sigma_11 - Sigma_12 Sigma_22^-1 Sigma_21, with Sigma_22^-1
    applied by device solves on the factor of the same call."""
    if with_variance and p.mode != "dense":
        raise ValueError("conditional variance is available in dense mode only")
    coords = _coords_of(p.known)
    n = len(p.known)
    nb = min(p.tile_size(), n)
    radius = _radius_of(p.known)
    h = _handle_for(coords, nb, p.max_rank, 1, radius)
    uxy = _coords_of(p.unknown)
    acc = p.accuracy if p.mode == "tlr" else None
    if not with_variance:
        return h.predict(np.asarray(p.z, dtype=float), uxy, p.theta, acc)
    # one device call: factor, mean, S22^-1 S21 (m right-hand sides), S11 - S12 (.)
    return h.predict_var(np.asarray(p.z, dtype=float), uxy, p.theta, acc)


# ------------------------------------------------------ component entry points
def bessel_k(nu: float, x) -> np.ndarray:
    """K_nu(x) evaluated on the device (kernels.py:160-174)."""
    lib = _lib.load()
    x = np.ascontiguousarray(np.atleast_1d(x), dtype=np.float64)
    out = np.empty_like(x)
    rc = lib.tlrb_bessel_k(float(nu), dptr(x), x.size, dptr(out), 0)
    if rc:
        raise ValueError(f"tlrb_bessel_k failed ({rc})")
    return out


def matern_block(rows_xy, cols_xy, p: MaternParams, radius: float = 0.0) -> np.ndarray:
    """Dense kernel block on the device (kernels.py:494-530, no nugget);
    radius > 0: great-circle distance, points as (lon, lat) degrees."""
    lib = _lib.load()
    a = np.ascontiguousarray(rows_xy, dtype=np.float64)
    b = np.ascontiguousarray(cols_xy, dtype=np.float64)
    out = np.empty((b.shape[0], a.shape[0]))  # column-major m x n == row-major n x m
    rc = lib.tlrb_matern_block_metric(dptr(a), a.shape[0], dptr(b), b.shape[0], p.theta1, p.theta2,
                                      p.theta3, float(radius), dptr(out), 0)
    if rc:
        raise ValueError(f"tlrb_matern_block failed ({rc})")
    return out.T.copy()


def compress_tile(a: np.ndarray, eps: float):
    """Device compression of one tile; returns (u, v) with a ~= u v^T
    (compression.py:39-51 contract)."""
    lib = _lib.load()
    a = np.asarray(a, dtype=np.float64)
    m, n = a.shape
    af = np.asfortranarray(a)
    k = np.zeros(1, np.int32)
    u = np.zeros(m * min(m, n))
    v = np.zeros(n * min(m, n))
    rc = lib.tlrb_compress_tile(dptr(af), m, n, float(eps), iptr(k), dptr(u), dptr(v), 0)
    if rc:
        raise ValueError(f"tlrb_compress_tile failed ({rc})")
    r = int(k[0])
    return (u[: m * r].reshape(r, m).T.copy(), v[: n * r].reshape(r, n).T.copy())


def potrf_tile(a: np.ndarray, tile_index: int = 0) -> np.ndarray:
    """Device Cholesky of one tile, lower factor (linalg.potrf_tile,
    linalg.py:36-45); raises NotPositiveDefiniteError(tile_index, pivot)."""
    lib = _lib.load()
    a = np.asarray(a, dtype=np.float64)
    n = a.shape[0]
    if a.ndim != 2 or a.shape[1] != n:
        raise ValueError(f"tile must be square, got {a.shape}")
    af = np.asfortranarray(a)
    out = np.zeros((n, n), order="F")
    piv = np.zeros(1, np.int32)
    rc = lib.tlrb_potrf_tile(dptr(af.ravel(order="K")), n, int(tile_index), out.ctypes.data_as(_lib._DP),
                             iptr(piv), 0)
    if rc == _lib.TLRB_ERR_NPD:
        raise NotPositiveDefiniteError(int(tile_index), int(piv[0]))
    if rc:
        raise ValueError(f"tlrb_potrf_tile failed ({rc})")
    return np.ascontiguousarray(out)


def launch_count() -> int:
    return int(_lib.load().tlrb_launch_count())
