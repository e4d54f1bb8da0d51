"""ctypes binding of the C ABI in include/aliasfft_b200.h.

The shared library is built in-tree (``paper_2011_05749_b200/libaliasfft_b200.so``)
by ``__graft_entry__.build()`` / ``make -C paper_2011_05749_b200/csrc``.  There is
no CPU fallback: every hot-path call goes through this library on a CUDA
device, and a missing library or device raises instead of degrading.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libaliasfft_b200.so")

AFFT_C64 = 0
AFFT_C128 = 1

AFFT_OK = 0
AFFT_EINVAL = -1
AFFT_EUNSUPPORTED = -2
AFFT_ECUDA = -3
AFFT_ENOMEM = -4

_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_INT = ctypes.c_int
_SZ = ctypes.c_size_t
_D = ctypes.c_double

# name -> (restype, argtypes); the list every test checks against the header.
SIGNATURES = {
    "afft_last_error": (ctypes.c_char_p, []),
    "afft_version": (_INT, []),
    "afft_bucketize": (_INT, [_P, _INT, _I64, _I64, _I64, _I64, _P, _I32, _P, _I64, _I64, _I64, _P]),
    "afft_build_graph": (_INT, [_P, _INT, _I64, _I64, _I64, _P, _I32, _P, _I32, _P, _P]),
    "afft_sumsq_parts": (_I32, [_I64, _INT]),
    "afft_sumsq": (_INT, [_P, _INT, _I64, _I64, _I64, _P, _P]),
    "afft_exact_thresholds": (_INT, [_P, _I32, _I64, _I64, _P, _P]),
    "afft_peel_exact": (
        _INT,
        [_I64, _I64, _P, _I32, _P, _P, _P, _P, _P, _P, _I32, _P, _P, _I32, _P, _P, _P, _P],
    ),
    "afft_peel_tree_exact": (
        _INT,
        [_I64, _I64, _P, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _I32, _P, _P, _P, _P, _P],
    ),
    "afft_classify_exact": (_INT, [_P, _P, _I64, _I64, _I64, ctypes.c_double, ctypes.c_double, _P, _P, _P, _P]),
    "afft_subtract": (_INT, [_P, _P, _I32, _P, _P, _I64, _I64, _P]),
    "afft_truncate": (_INT, [_P, _P, _P, _I32, _I64, _I32, _P, _P, _P, _P]),
    "afft_truncate_host": (_INT, [_P, _P, _I64, _I32, _P, _P, _P]),
    "afft_ffast_occupancy": (_INT, [_I64, _P, _I32, _P, _P]),
    "afft_ffast_workspace_size": (_SZ, [_I64, _INT, _I64, _P, _I32]),
    "afft_ffast": (
        _INT,
        [_P, _INT, _I64, _I64, _I64, _P, _I32, _I32, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P],
    ),
    "afft_node_energies": (_INT, [_P, _I32, _I64, _P, _P]),
    "afft_robust_thresholds": (_INT, [_P, _P, _I64, _I64, _I32, _P, _P, _P]),
    "afft_noisy_workspace_size": (_SZ, [_I64, _I64, _P, _I32, _I32, _I32]),
    "afft_singleton_workspace_size": (_SZ, [_I64, _I64, _I64, _I32, _I32]),
    "afft_singleton_search_noisy": (
        _INT, [_P, _P, _I64, _I64, _I64, _P, _I32, _I32, _I32, _P, _P, _P, _P, _P, _SZ, _P]),
    "afft_classify_noisy": (
        _INT, [_P, _P, _I64, _I64, _I64, _P, _I32, _I32, _I32, _P, _D, _D, _P, _P, _P, _P, _P,
               _SZ, _P]),
    "afft_peel_noisy": (
        _INT, [_I64, _I64, _P, _I32, _P, _I32, _I32, _I32, _P, _P, _P, _P, _P, _P, _P, _I32, _P,
               _P, _I32, _P, _P, _P, _P, _SZ, _P]),
    "afft_peel_noisy_sharded": (
        _INT, [_I64, _I64, _P, _I32, _P, _I32, _I32, _I32, _P, _P, _P, _P, _P, _P, _P, _I32, _P,
               _P, _I32, _P, _P, _P, _P, _SZ, _P, _P]),
    "afft_rffast_workspace_size": (_SZ, [_I64, _I64, _P, _I32, _I32, _I32]),
    "afft_rffast": (
        _INT, [_P, _INT, _I64, _I64, _I64, _P, _I32, _P, _I64, _I32, _I32, _P, _I32, _I32, _P, _P,
               _P, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "afft_small_la": (_INT, [_I32, _I32, _I32, _P, _P, _I32, _P, _P, _P, _P, _P, _P]),
    "afft_bucketize_table": (_INT, [_P, _INT, _I64, _I64, _I64, _I64, _P, _I32, _P, _I64, _I64,
                                    _I64, _P]),
    "afft_dt_collect": (_INT, [_P, _INT, _I64, _I64, _I64, _I64, _I32, _I32, _P, _P, _P]),
    "afft_dt_detect": (_INT, [_P, _I64, _I64, _I32, _I32, _I32, _P, _P, _P]),
    "afft_dt_locate": (_INT, [_P, _I64, _I32, _I32, _P, _P, _I32, _I64, _I64, _P, _P, _P]),
    "afft_dt_estimate": (_INT, [_P, _P, _I64, _I32, _I32, _P, _P, _I64, _I64, _P, _P, _P, _P]),
    "afft_dt_solve": (_INT, [_P, _P, _I64, _I64, _I32, _I32, _P, _P, _I32, _I32, _I64, _I64, _P,
                             _P, _P, _P]),
    "afft_dt_truncate": (_INT, [_P, _P, _P, _I64, _I64, _I32, _I32, _P, _P, _P, _P, _P, _P, _P]),
    "afft_sfft_dt_workspace_size": (_SZ, [_I64, _I64, _I64, _I32, _I32]),
    "afft_sfft_dt": (_INT, [_P, _INT, _I64, _I64, _I64, _I64, _I32, _I32, _I32, _I32, _P, _P, _P,
                            _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "afft_bucketize_rows": (_INT, [_P, _INT, _I64, _I64, _P, _I32, _P, _I64, _P, _P, _P]),
    "afft_alias_rows": (_INT, [_P, _I64, _I64, _P, _I32, _P, _I64, _P, _P, _P, _P]),
    "afft_active_indices": (_INT, [_P, _I64, _D, _P, _P, _P, _P]),
    "afft_selective_sums": (_INT, [_P, _INT, _I64, _I64, _P, _I64, _P, _P]),
    "afft_median": (_INT, [_P, _I32, _I64, _I64, _P, _P]),
    "afft_dsfft": (_INT, [_P, _INT, _I64, _I32, _P, _P, _P, _I64, _P, _P, _I32, _P, _P]),
    "afft_dsfft_batch": (_INT, [_P, _INT, _I64, _I64, _I64, _I32, _P, _P, _P, _I64, _P, _P, _I32,
                                _P, _P, _P]),
}

_lock = threading.Lock()
_lib = None


class LibraryNotBuilt(ImportError):
    """The CUDA library is missing: build it with __graft_entry__.build()."""


# afft_exchange_fn(ctx, part_score, part_t, count, stream) -> int
EXCHANGE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                               ctypes.c_int64, ctypes.c_void_p)


class SearchShardC(ctypes.Structure):
    """AfftSearchShard (include/aliasfft_b200.h)."""

    _fields_ = [("rank", ctypes.c_int32), ("world", ctypes.c_int32),
                ("exchange", EXCHANGE_FN), ("ctx", ctypes.c_void_p)]


class DsfftParams(ctypes.Structure):
    """AfftDsfftParams (include/aliasfft_b200.h)."""

    _fields_ = [
        ("theta", ctypes.c_double),
        ("mode", ctypes.c_int32),
        ("a_m", ctypes.c_int32),
        ("noise_std", ctypes.c_double),
        ("activity_floor", ctypes.c_double),
        ("c", ctypes.c_int32),
        ("m", ctypes.c_int32),
        ("anchors", ctypes.c_void_p),
        ("weights", ctypes.c_void_p),
        ("dt_shifts", ctypes.c_void_p),
        ("dt_shift_off", ctypes.c_void_p),
        ("full_classify", ctypes.c_int32),
    ]


def load():
    """Load (once) and return the ctypes handle; raises if the .so is missing."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise LibraryNotBuilt(
                    f"{LIB_PATH} not found; run `python -c 'import __graft_entry__ as g; g.build()'`"
                )
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


_PYENTRIES_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_pyentries.so")
_entries_fn = None


def entries_dict(pos: np.ndarray, val: np.ndarray) -> dict:
    """dict(zip(pos, val)) for int64 positions and complex128 values, built by the
    in-tree C helper csrc/pyentries.c (half the GIL time of the Python form; host-side
    presentation of results already computed, so without the helper the Python form
    builds the same dict)."""
    global _entries_fn
    pos = np.ascontiguousarray(pos, dtype=np.int64)
    val = np.ascontiguousarray(val, dtype=np.complex128)
    if _entries_fn is None:
        fn = False
        if os.path.exists(_PYENTRIES_PATH):
            fn = ctypes.PyDLL(_PYENTRIES_PATH).afft_py_entries
            fn.restype = ctypes.py_object
            fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
        _entries_fn = fn
    if _entries_fn is False:
        return dict(zip(pos.tolist(), val.tolist()))
    return _entries_fn(pos.ctypes.data, val.ctypes.data, int(pos.size))


def check(status: int, what: str) -> None:
    """Map a C status to the reference's exception classes."""
    if status == AFFT_OK:
        return
    msg = load().afft_last_error().decode(errors="replace")
    text = f"{what}: {msg}"
    if status == AFFT_EINVAL:
        raise ValueError(text)
    if status == AFFT_EUNSUPPORTED:
        from .peeling import UnsupportedSizeError

        raise UnsupportedSizeError(text)
    if status == AFFT_ENOMEM:
        raise MemoryError(text)
    raise RuntimeError(text)


def host_f64(values) -> ctypes.Array:
    vals = [float(v) for v in values]
    return (ctypes.c_double * max(1, len(vals)))(*vals)


def host_i64(values) -> tuple[ctypes.Array, int]:
    """A host int64 array for the small plan arguments (factors, shifts)."""
    arr = np.ascontiguousarray(np.asarray(list(values), dtype=np.int64))
    buf = (ctypes.c_int64 * max(1, arr.size))(*arr.tolist())
    return buf, int(arr.size)
