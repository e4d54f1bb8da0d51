"""CPU check of the device sFFT-DT code (csrc/smallla.cuh, csrc/oneshot_core.cuh).

The kernel sources are compiled for the host with g++ (tests/native/build.py) and
compared with numpy / the oracle: small complex LA against numpy.linalg, and the
per-bucket locate + pursuit against oracle/oneshot.py on real measurement rows.
"""

import ctypes
import zlib

import numpy as np
import pytest

from native.build import host_lib
from oracle import oneshot as od
from paper_2011_05749_b200.signals import generate_test_case

P = ctypes.c_void_p
VAR = {"dt1": 1, "dt2": 2, "dt3": 3}


def ptr(a):
    return a.ctypes.data_as(P)


def test_small_la_matches_numpy():
    lib = host_lib()
    rng = np.random.default_rng(0)
    for trial in range(200):
        m, n = int(rng.integers(1, 9)), int(rng.integers(1, 9))
        A = rng.normal(size=(m, n)) + 1j * rng.normal(size=(m, n))
        if trial % 3 == 0 and min(m, n) > 1:
            A[:, -1] = 2 * A[:, 0]
        a = np.ascontiguousarray(A)
        s = np.zeros(min(m, n))
        lib.t_singular_values(m, n, ptr(a), ptr(s))
        sv = np.linalg.svd(A, compute_uv=False)
        assert np.max(np.abs(s - sv)) <= 1e-13 * sv[0]
        pv = np.zeros((n, m), complex)
        lib.t_pinv(m, n, ptr(a), ctypes.c_double(1e-15), ptr(pv))
        ref = np.linalg.pinv(A)
        assert np.max(np.abs(pv - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))
        if m >= n:
            y = rng.normal(size=m) + 1j * rng.normal(size=m)
            x = np.zeros(n, complex)
            rank = lib.t_lstsq(m, n, ptr(a), ptr(y), ptr(x), ptr(np.zeros(n)))
            xr, _, rk, _ = np.linalg.lstsq(A, y, rcond=None)
            assert rank == rk
            assert np.max(np.abs(x - xr)) <= 1e-12 * max(1.0, np.max(np.abs(xr)))
        if m == n:
            lam = np.zeros(n, complex)
            lib.t_eigvals(n, ptr(a), ptr(lam))
            ev = np.linalg.eigvals(A)
            assert max(min(abs(l - e) for e in ev) for l in lam) <= 1e-12 * max(abs(ev))


def _case(n, k, snr, b, p, seed_trial=0):
    tag = "exact" if snr == "exact" else f"{float(snr):.9g}"
    seed = zlib.crc32(f"{n}|{k}|{tag}|0|{seed_trial}".encode())
    x = generate_test_case(n, k, snr, seed).signal
    rsh = od.random_shifts(n, p, seed)
    rows = od.measurement_rows(x, b, 4, rsh)
    return rows, rsh, od.vote(rows, k, 4)


@pytest.mark.parametrize("variant", ["dt1", "dt2", "dt3"])
@pytest.mark.parametrize("cfg", [(1 << 14, 16, "exact", 512, 12), (1 << 16, 16, 20.0, 2048, 12),
                                 (1 << 18, 200, "exact", 256, 12)])
def test_bucket_solve_matches_oracle(variant, cfg):
    n, k, snr, b, p = cfg
    rows, rsh, counts = _case(n, k, snr, b, p)
    lib = host_lib()
    sh = np.ascontiguousarray(np.array(rsh, dtype=np.int64))
    checked = 0
    for bucket in np.flatnonzero(counts):
        a = int(counts[bucket])
        row = np.ascontiguousarray(rows[bucket])
        cands = od.locate(row, 4, a, variant, int(bucket), b, n)
        pos = np.zeros(4, np.int64)
        nl = lib.t_locate(ptr(row), 4, a, VAR[variant], int(bucket), b, n, ptr(pos))
        if cands is None:
            assert nl == -1
            continue
        assert list(pos[:nl]) == list(cands), (variant, bucket, a)
        want_p, want_v = od.pursue(row[12:], rsh, cands, b, n)
        vals = np.zeros(4, complex)
        cnt = lib.t_solve_bucket(ptr(row), 4, p, ptr(sh), a, VAR[variant], int(bucket), b, n,
                                 ptr(pos), ptr(vals))
        # same position -> value map (list order can differ on exact correlation ties)
        got = dict(zip(pos[:cnt].tolist(), vals[:cnt].tolist()))
        assert set(got) == set(want_p), (variant, bucket)
        for f, v in zip(want_p, want_v):
            assert abs(got[f] - v) <= 1e-9
        checked += 1
    assert checked > 0
