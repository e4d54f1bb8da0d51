"""Oracle: R-FFAST (noisy peeling) in numpy.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Restates
/root/reference/pkg/src/aliasfft/peeling.py:218-267 (singleton search,
classify_noisy), 335-358 (robust/noisy thresholds) and the noisy branch of
peel_decode (270-313) on a (nodes, R) residual matrix.  The per-node search is
vectorised over candidates exactly as the reference evaluates it, so scores are
bit-identical to the reference's.
"""

from __future__ import annotations

import numpy as np

from .ffast import MULTI, RESOLVED, SINGLE, ZERO, tone_rows


def wrap(p):
    """((p + pi) mod 2pi) - pi  (peeling.py:218-219)."""
    return (p + np.pi) % (2.0 * np.pi) - np.pi


def thresholds(energies, r: int, scale=None):
    """(T0, T1) from the median energy (peeling.py:335-351)."""
    e = np.asarray(energies, dtype=float)
    s = e if scale is None else np.asarray(scale, dtype=float)
    sigma = np.sqrt(max(float(np.median(e)), 0.0) / r)
    floor = 1e-8 * np.sqrt(float(s.max(initial=0.0)))
    base = sigma * np.sqrt(r)
    return max(1.5 * base, floor), max(2.5 * base, floor)


def node_energies(values: np.ndarray) -> np.ndarray:
    """||vec||^2 per node row (peeling.py:355-357)."""
    return np.array([float(np.linalg.norm(row) ** 2) for row in values])


def search(y, index: int, b: int, n: int, c: int, m: int, weights, shifts):
    """Exhaustive residue-class candidate scan + 1-column LS (peeling.py:222-250).

    Returns (f0, value, resnorm).
    """
    y = np.asarray(y, dtype=np.complex128)
    L = n // b
    cands = (index + b * np.arange(L, dtype=np.int64)) % n
    score = np.zeros(L)
    for j in range(c):
        seg = y[j * m:(j + 1) * m]
        d = np.angle(seg[1:] * np.conj(seg[:-1]))
        d = d[0] + wrap(d - d[0])
        est = float(np.dot(weights, d))
        score += wrap(est - (-2.0 * np.pi * (((1 << j) * cands) % n) / n)) ** 2
    f0 = int(cands[int(np.argmin(score))])
    atom = tone_rows(f0, shifts, n)[:, None]
    x, *_ = np.linalg.lstsq(atom, y, rcond=None)
    return f0, complex(x[0]), float(np.linalg.norm(atom @ x - y))


def peel_noisy(values: np.ndarray, factors, n: int, c: int, m: int, weights, shifts, t0: float,
               t1: float, max_rounds: int):
    """Noisy synchronous peeling on (nodes, R): dict like oracle.ffast.peel_exact."""
    factors = [int(b) for b in factors]
    res = np.array(values, dtype=np.complex128, copy=True)
    cyc = np.repeat(np.arange(len(factors)), factors)
    base = np.concatenate(([0], np.cumsum(factors)[:-1])).astype(np.int64)
    index = np.arange(len(res)) - base[cyc]
    state = np.zeros(len(res), dtype=np.int8)
    f0 = np.full(len(res), -1, dtype=np.int64)
    value = np.zeros(len(res), dtype=np.complex128)
    dirty = np.ones(len(res), dtype=bool)  # classification is a pure function of the residual
    recovered: dict[int, complex] = {}
    rounds = 0
    for _ in range(max_rounds):
        rounds += 1
        found: dict[int, complex] = {}
        for g in range(len(res)):
            if state[g] in (RESOLVED, ZERO):
                continue
            if dirty[g]:
                dirty[g] = False
                if np.linalg.norm(res[g]) <= t0:
                    state[g] = ZERO
                    continue
                f, v, rn = search(res[g], int(index[g]), factors[cyc[g]], n, c, m, weights, shifts)
                if rn <= t1:
                    state[g], f0[g], value[g] = SINGLE, f, v
                else:
                    state[g] = MULTI
            if state[g] == SINGLE and f0[g] not in recovered and f0[g] not in found:
                found[int(f0[g])] = complex(value[g])
                state[g] = RESOLVED
        if not found:
            break
        for f, v in found.items():
            for ci, b in enumerate(factors):
                g = base[ci] + f % b
                res[g] = res[g] - v * tone_rows(f, shifts, n)
                dirty[g] = True
        recovered.update(found)
    return {"recovered": recovered, "rounds": rounds,
            "unresolved": int(np.sum(state == MULTI)), "state": state, "residual": res}
