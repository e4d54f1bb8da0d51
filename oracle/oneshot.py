"""Oracle: sFFT-DT1/2/3 in numpy.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Restates
/root/reference/pkg/src/aliasfft/oneshot.py:27-289 and smallnum.py:54-142 over
a (b, 3*a_m + p) measurement-row matrix instead of per-bucket dict objects:
columns 0..3a_m-1 hold the structured shifts -a_m..2a_m-1, the rest the p
seeded random shifts.  LAPACK (numpy.linalg) does the small solves, as in the
reference.
"""

from __future__ import annotations

import numpy as np

from .ffast import bucket_values

TIE_QUANTUM = 1e-12  # oneshot.py:24
SP_MAX_ITERS = 10    # oneshot.py:23


def structured_shifts(a_m: int) -> list[int]:
    """-a_m .. 2a_m-1 (oneshot.py:81-83)."""
    return list(range(-a_m, 2 * a_m))


def random_shifts(n: int, p: int, seed: int) -> list[int]:
    """rng.choice(n, p, replace=False) with the config seed (oneshot.py:93-94)."""
    return [int(t) for t in np.random.default_rng(seed).choice(n, size=p, replace=False)]


def validate(n: int, b: int, a_m: int, p: int, variant: str) -> None:
    """OneShotConfig.validate (oneshot.py:48-60)."""
    if variant not in ("dt1", "dt2", "dt3"):
        raise ValueError(variant)
    if not 1 <= a_m <= 4 or b < 1 or n % b:
        raise ValueError("bad config")
    if p < a_m * np.log10(max(n // b, 1)):
        raise ValueError("p below the measurement floor")


def measurement_rows(x, b: int, a_m: int, rshifts) -> np.ndarray:
    """(b, 3a_m + p) bucket values at the structured then random shifts (86-106)."""
    shifts = structured_shifts(a_m) + list(rshifts)
    return bucket_values(x, b, shifts).T


def hankel(row, a_m: int, size: int, start: int = 0) -> np.ndarray:
    return np.array([[row[a_m + start + r + c] for c in range(size)] for r in range(size)],
                    dtype=np.complex128)


def vote(rows: np.ndarray, k: int, a_m: int) -> np.ndarray:
    """detect_sparsity (oneshot.py:116-140): global top-k of quantised Hankel sigmas."""
    b = rows.shape[0]
    counts = np.zeros(b, dtype=int)
    if k <= 0:
        return counts
    sig = np.stack([np.linalg.svd(hankel(r, a_m, a_m), compute_uv=False) for r in rows])
    flat = sig.ravel()
    bucket = np.repeat(np.arange(b), a_m)
    slot = np.tile(np.arange(a_m), b)
    q = np.round(flat / TIE_QUANTUM).astype(np.int64)
    chosen = np.lexsort((slot, bucket, -q))[: min(k, flat.size)]
    np.add.at(counts, bucket[chosen], 1)
    return counts


def unit_root(f, n: int, e=1):
    prod = (np.asarray(e, dtype=np.int64) * np.asarray(f, dtype=np.int64)) % n
    return np.exp(-2j * np.pi * prod / n)


def snap(z: complex, bucket: int, b: int, n: int) -> int:
    """_snap_to_grid (oneshot.py:150-158)."""
    step = n // b
    f_est = (-np.angle(z) * n / (2.0 * np.pi)) % n
    d = (f_est - bucket) / b
    j = int(np.floor(d + 0.5))
    if abs(d - np.floor(d) - 0.5) < 1e-12:
        j = int(np.floor(d))
    return (bucket + (j % step) * b) % n


def lstsq_solution(a, y):
    x, *_ = np.linalg.lstsq(a, y, rcond=None)
    return x


def pencil_roots(full: np.ndarray, a: int):
    """pencil_eigenvalues(full[:, :-1], full[:, 1:], a).values (smallnum.py:110-142)."""
    sv = np.linalg.svd(full, compute_uv=False)
    rank = min(a, int(np.sum(sv > sv[0] * 1e-10)))
    if rank == 0:
        return np.zeros(0, dtype=np.complex128)
    _, _, vh = np.linalg.svd(full)
    basis = vh[:rank, :]
    return np.conj(np.linalg.eigvals(basis[:, 1:] @ np.linalg.pinv(basis[:, :-1])))


def locate(row, a_m: int, a: int, variant: str, bucket: int, b: int, n: int):
    """Candidate positions, or None (oneshot.py:161-200)."""
    if a < 1:
        return []
    step = n // b
    if variant == "dt3":
        full = np.array([[row[a_m + r - c] for c in range(a + 1)] for r in range(a + 1)],
                        dtype=np.complex128)
        roots = pencil_roots(full, a)
        if roots.size == 0 or not np.all(np.isfinite(roots)):
            return None
        return sorted({snap(z, bucket, b, n) for z in roots})
    coeffs = lstsq_solution(hankel(row, a_m, a),
                            -np.array([row[a_m + a + r] for r in range(a)], dtype=np.complex128))
    if not np.all(np.isfinite(coeffs)):
        return None
    if variant == "dt1":
        if a == 1:
            roots = np.array([-coeffs[0]])
        elif a == 2:
            s = np.sqrt(coeffs[1] * coeffs[1] - 4.0 * coeffs[0] + 0j)
            roots = np.array([(-coeffs[1] - s) / 2.0, (-coeffs[1] + s) / 2.0])
        else:
            roots = np.roots(np.concatenate(([1.0 + 0j], coeffs[::-1])))
        return sorted({snap(z, bucket, b, n) for z in roots})
    cands = (bucket + b * np.arange(step)) % n
    pv = np.polyval(np.concatenate(([1.0 + 0j], coeffs[::-1])), unit_root(cands, n))
    best = np.argsort(np.abs(pv), kind="stable")[: min(a, step)]
    return sorted(int(cands[j]) for j in best)


def pursue(rand_vals, rshifts, candidates, b: int, n: int):
    """estimate_values (oneshot.py:203-257): (positions, values)."""
    y = np.asarray(rand_vals, dtype=np.complex128)
    shifts = np.asarray(rshifts, dtype=np.int64)
    candidates = sorted(set(int(f) for f in candidates))
    if not candidates or np.linalg.norm(y) == 0.0:
        return [], []
    freqs: list[int] = []
    for f in candidates:
        for g in (f, (f + b) % n, (f - b) % n):
            if g not in freqs:
                freqs.append(g)
    fa = np.array(freqs, dtype=np.int64)
    atoms = unit_root(fa[None, :], n, shifts[:, None])
    want = min(len(candidates), len(freqs), len(shifts))
    tol = 1e-10 * max(1.0, float(np.linalg.norm(y)))

    def fit(sup):
        coef = lstsq_solution(atoms[:, sup], y)
        return coef, float(np.linalg.norm(y - atoms[:, sup] @ coef))

    sup = np.argsort(-np.abs(atoms.conj().T @ y), kind="stable")[:want]
    coef, res = fit(sup)
    best = (sup, coef, res)
    for _ in range(SP_MAX_ITERS):
        if best[2] <= tol:
            break
        r = y - atoms[:, best[0]] @ best[1]
        fresh = np.argsort(-np.abs(atoms.conj().T @ r), kind="stable")[:want]
        merged = np.union1d(best[0], fresh)
        coef_m, _ = fit(merged)
        pruned = np.sort(merged[np.argsort(-np.abs(coef_m), kind="stable")[:want]])
        coef, res = fit(pruned)
        if res >= best[2]:
            break
        best = (pruned, coef, res)
    return [int(fa[j]) for j in best[0]], [complex(v) for v in best[1]]


def truncate(entries: dict, k: int) -> dict:
    ranked = sorted(entries.items(), key=lambda kv: (-abs(kv[1]), kv[0]))
    return dict(ranked[:k])


def sfft_dt(x, k: int, b: int, a_m: int = 4, p: int = 12, variant: str = "dt3", seed: int = 0):
    """Full pipeline (oneshot.py:266-289): returns (truncated, entries, counts)."""
    x = np.asarray(x, dtype=np.complex128)
    n = x.size
    validate(n, b, a_m, p, variant)
    rsh = random_shifts(n, p, seed)
    rows = measurement_rows(x, b, a_m, rsh)
    counts = vote(rows, k, a_m)
    entries: dict[int, complex] = {}
    for bucket in range(b):
        a = int(counts[bucket])
        if a == 0:
            continue
        cands = locate(rows[bucket], a_m, a, variant, bucket, b, n)
        if cands is None:
            continue
        pos, vals = pursue(rows[bucket, 3 * a_m:], rsh, cands, b, n)
        for f, v in zip(pos, vals):
            entries[f] = v
    return truncate(entries, k), entries, counts
