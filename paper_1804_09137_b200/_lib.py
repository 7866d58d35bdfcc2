"""ctypes binding of libtlrb200.so (the C ABI declared in include/tlrb200.h).

The product path has no CPU fallback: if the shared library is missing or
fails to load, every entry point raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libtlrb200.so"

TLRB_OK, TLRB_ERR_NPD, TLRB_ERR_ARG, TLRB_ERR_CUDA = 0, 1, 2, 3
TLRB_BACKEND_AUTO, TLRB_BACKEND_NCCL, TLRB_BACKEND_LOOPBACK = 0, 1, 2


class TlrbStats(C.Structure):
    _fields_ = [
        ("ms_generate", C.c_double),
        ("ms_compress", C.c_double),
        ("ms_factor", C.c_double),
        ("ms_solve", C.c_double),
        ("ms_total", C.c_double),
        ("ms_device", C.c_double),
        ("flops", C.c_double),
        ("bytes", C.c_double),
        ("stored_reals", C.c_int64),
        ("kernel_launches", C.c_int64),
        ("max_rank", C.c_int32),
        ("mean_rank", C.c_double),
        ("sketch_retries", C.c_int32),
        ("jacobi_max_sweeps", C.c_int32),
        ("t_roof_ms", C.c_double),
        ("arena_peak_bytes", C.c_int64),
        ("panel_peak_bytes", C.c_int64),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


_lib = None

# (name, restype, argtypes) — mirrors include/tlrb200.h
_DP = C.POINTER(C.c_double)
_IP = C.POINTER(C.c_int32)
SIGNATURES = [
    ("tlrb_create", C.c_void_p, [_DP, C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _IP]),
    ("tlrb_destroy", None, [C.c_void_p]),
    ("tlrb_nccl_unique_id", C.c_int32, [C.c_char_p, C.c_int32]),
    ("tlrb_create_dist", C.c_void_p, [_DP, C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                      C.c_int32, C.c_int32, C.c_char_p, _IP]),
    ("tlrb_set_metric", C.c_int32, [C.c_void_p, C.c_double]),
    ("tlrb_loglik", C.c_int32, [C.c_void_p, _DP, C.c_double, C.c_double, C.c_double, C.c_double,
                                C.c_double, _DP, _DP, _DP, C.POINTER(TlrbStats)]),
    ("tlrb_loglik_device", C.c_int32, [C.c_void_p, C.c_void_p, C.c_double, C.c_double, C.c_double,
                                       C.c_double, C.c_double, _DP, _DP, _DP, C.POINTER(TlrbStats)]),
    ("tlrb_factorize", C.c_int32, [C.c_void_p, C.c_double, C.c_double, C.c_double, C.c_double,
                                   C.c_double]),
    ("tlrb_apply_factor", C.c_int32, [C.c_void_p, _DP, _DP]),
    ("tlrb_solve", C.c_int32, [C.c_void_p, _DP, _DP]),
    ("tlrb_predict", C.c_int32, [C.c_void_p, _DP, _DP, C.c_int64, C.c_double, C.c_double, C.c_double,
                                 C.c_double, C.c_double, _DP]),
    ("tlrb_predict_var", C.c_int32, [C.c_void_p, _DP, _DP, C.c_int64, C.c_double, C.c_double, C.c_double,
                                     C.c_double, C.c_double, _DP, _DP]),
    ("tlrb_rank_map", C.c_int32, [C.c_void_p, _IP, C.c_int32, _IP]),
    ("tlrb_last_error", C.c_int32, [C.c_void_p, _IP, _IP, C.c_char_p, C.c_int32]),
    ("tlrb_bessel_k", C.c_int32, [C.c_double, _DP, C.c_int64, _DP, C.c_int32]),
    ("tlrb_matern_block", C.c_int32, [_DP, C.c_int64, _DP, C.c_int64, C.c_double, C.c_double,
                                      C.c_double, _DP, C.c_int32]),
    ("tlrb_matern_block_metric", C.c_int32, [_DP, C.c_int64, _DP, C.c_int64, C.c_double, C.c_double,
                                             C.c_double, C.c_double, _DP, C.c_int32]),
    ("tlrb_compress_tile", C.c_int32, [_DP, C.c_int32, C.c_int32, C.c_double, _IP, _DP, _DP, C.c_int32]),
    ("tlrb_potrf_tile", C.c_int32, [_DP, C.c_int32, C.c_int32, _DP, _IP, C.c_int32]),
    ("tlrb_launch_count", C.c_int64, []),
    ("tlrb_profile_enable", C.c_int32, [C.c_int32]),
    ("tlrb_profile_mask", C.c_int32, [C.c_uint32]),
    ("tlrb_profile_read", C.c_int32, [C.c_int32, C.c_char_p, C.c_int32, _DP, _DP, _DP,
                                      C.POINTER(C.c_int64)]),
    ("tlrb_profile_busy", C.c_int32, [C.c_int32, _DP]),
    ("tlrb_create_group", C.c_void_p, [_DP, C.c_int64, C.c_int32, C.c_int32, _IP, C.c_int32, C.c_int32,
                                       C.c_int32, C.c_int32, _IP]),
    ("tlrb_group_size", C.c_int32, [C.c_void_p]),
    ("tlrb_member_stats", C.c_int32, [C.c_void_p, C.c_int32, C.c_void_p]),
    ("tlrb_set_peaks", C.c_int32, [C.c_double, C.c_double]),
]


def load():
    """Load libtlrb200.so (raises if it is absent: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("TLRB200_LIB", LIB_PATH))
    if not path.exists():
        raise RuntimeError(f"libtlrb200.so not found at {path}; run __graft_entry__.build() "
                           "(the B200 path has no CPU fallback)")
    lib = C.CDLL(str(path))
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


KERNEL_CLASSES = ("gen_tiles", "dgemm_vbatch", "trsm_vbatch", "potrf_block", "qr_householder",
                  "jacobi_svd", "sumsq", "copy", "unused", "reduce", "cross_gemv")


def profile_enable(on: bool = True, classes=None):
    """Reset and (de)activate the per-launch CUDA-event profiler; `classes`
    (names) restricts it to those kernel classes."""
    lib = load()
    mask = 0xFFFFFFFF if classes is None else sum(1 << KERNEL_CLASSES.index(c) for c in classes)
    lib.tlrb_profile_mask(mask)
    lib.tlrb_profile_enable(1 if on else 0)


def profile_read() -> dict:
    """{kernel class: {ms, flops, bytes, launches}} since profile_enable()."""
    lib = load()
    out = {}
    for cls in range(11):
        name = C.create_string_buffer(64)
        v = np.zeros(3)
        cnt = C.c_int64(0)
        lib.tlrb_profile_read(cls, name, 64, dptr(v[0:]), dptr(v[1:]), dptr(v[2:]), C.byref(cnt))
        busy = np.zeros(1)
        lib.tlrb_profile_busy(cls, dptr(busy))
        out[name.value.decode()] = {"ms": float(v[0]), "flops": float(v[1]), "bytes": float(v[2]),
                                    "launches": int(cnt.value), "busy_ms": float(busy[0])}
    return out


def profile_busy_all() -> float:
    """Union of every profiled launch interval since profile_enable() (ms)."""
    busy = np.zeros(1)
    load().tlrb_profile_busy(-1, dptr(busy))
    return float(busy[0])


def dptr(a: np.ndarray):
    return a.ctypes.data_as(_DP)


def iptr(a: np.ndarray):
    return a.ctypes.data_as(_IP)
