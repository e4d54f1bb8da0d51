"""Oracle: bucketization and exact-mode peeling (FFAST) in numpy.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Array-based restatement of
/root/reference/pkg/src/aliasfft/bucketize.py:83-106 and peeling.py:169-332:
the graph is a (nodes, R) residual matrix with a parallel state vector instead
of BucketNode objects; classification of a round is vectorised, harvesting and
subtraction keep the reference's sequential order.
"""

from __future__ import annotations

import numpy as np

UNKNOWN, ZERO, SINGLE, MULTI, RESOLVED = 0, 1, 2, 3, 4


def bucket_values(x, b: int, shifts) -> np.ndarray:
    """(R, b) bucket values: fft(x[(j*L - tau) mod n]) / b  (bucketize.py:91-99)."""
    x = np.asarray(x, dtype=np.complex128)
    n = x.size
    if b < 1 or n % b:
        raise ValueError(f"bucket count {b} does not divide {n}")
    j = np.arange(b, dtype=np.int64) * (n // b)
    idx = (j[None, :] - np.asarray(list(shifts), dtype=np.int64)[:, None]) % n
    return np.fft.fft(x[idx], axis=1) / b


def graph_values(x, factors, shifts) -> np.ndarray:
    """(sum factors, R) node measurements, cycles in plan order (peeling.py:169-178)."""
    return np.concatenate([bucket_values(x, b, shifts).T for b in factors], axis=0)


def exact_eps(x) -> float:
    """1e-6 * ||x||_2 / sqrt(n)  (peeling.py:316-318)."""
    x = np.asarray(x, dtype=np.complex128)
    return 1e-6 * float(np.linalg.norm(x)) / np.sqrt(x.size)


def tone_rows(f: int, shifts, n: int) -> np.ndarray:
    """exp(-2j*pi*((tau*f) mod n)/n) over the shift list (peeling.py:181-183)."""
    prod = (np.asarray(list(shifts), dtype=np.int64) * int(f)) % n
    return np.exp(-2j * np.pi * prod / n)


def classify_rows(res: np.ndarray, index: np.ndarray, b: np.ndarray, n: int, eps0: float,
                  epsr: float):
    """Vectorised classify_exact (peeling.py:193-215) for rows of (r0, r1, r2).

    Returns (state, f0) with f0 = -1 where not SINGLE.
    """
    norm = np.sqrt(np.sum(res.real**2, axis=1) + np.sum(res.imag**2, axis=1))
    r0, r1, r2 = res[:, 0], res[:, 1], res[:, 2]
    state = np.full(len(res), MULTI, dtype=np.int8)
    state[norm <= eps0] = ZERO
    f0 = np.full(len(res), -1, dtype=np.int64)
    live = state == MULTI
    with np.errstate(divide="ignore", invalid="ignore"):
        ok = live & (np.minimum(np.abs(r0), np.abs(r1)) > eps0)
        q1 = np.where(ok, r1 / np.where(ok, r0, 1.0), 0.0)
        q2 = np.where(ok, r2 / np.where(ok, r1, 1.0), 0.0)
        ok &= np.abs(q1 - q2) <= epsr
        dec = np.round(np.angle(q1) * (-n / (2.0 * np.pi)))
    cand = np.where(ok, dec, 0).astype(np.int64) % n
    single = ok & (cand % b == index)
    state[single] = SINGLE
    f0[single] = cand[single]
    return state, f0


def peel_exact(values: np.ndarray, factors, n: int, eps0: float, epsr: float,
               max_rounds: int, shifts=(0, 1, 2)):
    """Synchronous exact peeling (peeling.py:270-313) on a (nodes, 3) matrix.

    Returns dict(recovered in insertion order, rounds, unresolved, state, residual).
    """
    factors = [int(b) for b in factors]
    res = np.array(values, dtype=np.complex128, copy=True)
    cyc = np.repeat(np.arange(len(factors)), factors)
    base = np.concatenate(([0], np.cumsum(factors)[:-1])).astype(np.int64)
    index = np.arange(len(res)) - base[cyc]
    bvec = np.asarray(factors, dtype=np.int64)[cyc]
    state = np.zeros(len(res), dtype=np.int8)
    f0 = np.full(len(res), -1, dtype=np.int64)
    value = np.zeros(len(res), dtype=np.complex128)
    recovered: dict[int, complex] = {}
    rounds = 0
    for _ in range(max_rounds):
        rounds += 1
        live = (state != RESOLVED) & (state != ZERO)
        st, fz = classify_rows(res[live], index[live], bvec[live], n, eps0, epsr)
        state[live] = st
        hit = np.flatnonzero(live)[st == SINGLE]
        f0[hit] = fz[st == SINGLE]
        value[hit] = res[hit, 0]
        found: dict[int, complex] = {}
        for g in hit:  # ascending node order == (cycle, index) order
            f = int(f0[g])
            if f not in recovered and f not in found:
                found[f] = complex(value[g])
                state[g] = RESOLVED
        if not found:
            break
        for f, v in found.items():
            for c, b in enumerate(factors):
                g = base[c] + f % b
                res[g] = res[g] - v * tone_rows(f, shifts, n)
        recovered.update(found)
    unresolved = int(np.sum(state == MULTI))
    return {"recovered": recovered, "rounds": rounds, "unresolved": unresolved,
            "state": state, "residual": res, "f0": f0}


def truncate(entries: dict, k: int) -> dict:
    """k largest |v|, ties to the smaller position (oneshot.py:260-263)."""
    ranked = sorted(entries.items(), key=lambda kv: (-abs(kv[1]), kv[0]))
    return dict(ranked[:k])


def ffast(x, k: int, factors, max_rounds: int | None = None):
    """ffast with an explicit plan (peeling.py:321-332): returns (truncated, decode dict)."""
    x = np.asarray(x, dtype=np.complex128)
    n = x.size
    vals = graph_values(x, factors, (0, 1, 2))
    eps = exact_eps(x)
    out = peel_exact(vals, factors, n, eps, eps, max_rounds or k + 4)
    return (truncate(out["recovered"], k) if k else {}), out
