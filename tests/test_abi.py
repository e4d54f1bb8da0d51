"""The C-ABI library loads and exports exactly what include/aliasfft_b200.h declares.

No compute calls here (no GPU needed): symbol presence, ctypes signatures, and
that the product fails loudly instead of falling back to the CPU.
"""

import os
import re

import numpy as np
import pytest
import torch

from paper_2011_05749_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                      "aliasfft_b200.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(afft_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_functions():
    names = header_functions()
    assert "afft_ffast" in names and "afft_bucketize" in names


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    for name in header_functions():
        assert hasattr(lib, name), name


def test_ctypes_table_covers_header():
    assert sorted(_lib.SIGNATURES) == header_functions()


def test_version_and_host_only_queries():
    lib = _lib.load()
    assert lib.afft_version() >= 1
    assert lib.afft_sumsq_parts(2097024, _lib.AFFT_C64) == 256
    fb, nc = _lib.host_i64([127, 128, 129])
    assert lib.afft_ffast_workspace_size(2097024, _lib.AFFT_C64, 4, fb, nc) > 0
    bad, nb = _lib.host_i64([127, 5])
    assert lib.afft_ffast_workspace_size(2097024, _lib.AFFT_C64, 4, bad, nb) == 0


def test_error_mapping_without_launch():
    lib = _lib.load()
    # null signal pointer -> EINVAL, reported through afft_last_error, no kernel launched
    sb, ns = _lib.host_i64([0])
    rc = lib.afft_bucketize(None, 0, 8, 1, 8, 4, sb, ns, None, 4, 4, 1, None)
    assert rc == _lib.AFFT_EINVAL
    with pytest.raises(ValueError):
        _lib.check(rc, "bucketize")


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    from paper_2011_05749_b200 import bucketize, ffast
    from paper_2011_05749_b200._device import NoCudaDevice

    with pytest.raises(NoCudaDevice):
        bucketize(np.zeros(8, dtype=complex), 4, 0)
    with pytest.raises(NoCudaDevice):
        ffast(np.zeros(20, dtype=complex), 2, plan=None)


def test_truncate_host_matches_numpy_order():
    """afft_truncate_host (host only, no device) keeps truncate_spectrum's order
    (oneshot.py:260-263): the k largest |v| (numpy's abs), ties to the smaller position —
    checked against a numpy lexsort, with exact magnitude ties forced in."""
    import ctypes

    import numpy as np

    from paper_2011_05749_b200 import _lib

    rng = np.random.default_rng(5)
    for count, k in ((0, 4), (1, 1), (50, 10), (1000, 1000), (4600, 4096), (300, 400)):
        pos = rng.permutation(1 << 20)[:count].astype(np.int64)
        val = rng.normal(size=count) + 1j * rng.normal(size=count)
        if count > 8:  # exact ties: equal magnitudes at different positions
            val[1::7] = val[0]
            val[2::9] = val[0].conjugate()
        op = np.empty(max(1, min(count, k)), dtype=np.int64)
        ov = np.empty(max(1, min(count, k)), dtype=np.complex128)
        cnt = ctypes.c_int64(-1)
        rc = _lib.load().afft_truncate_host(pos.ctypes.data, val.ctypes.data, count, k,
                                            op.ctypes.data, ov.ctypes.data, ctypes.byref(cnt))
        assert rc == 0
        order = np.lexsort((pos, -np.abs(val)))[:k]
        assert cnt.value == len(order)
        assert op[: cnt.value].tolist() == pos[order].tolist()
        assert np.array_equal(ov[: cnt.value], val[order])
