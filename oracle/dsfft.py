"""Oracle: DSFFT binary-tree search in numpy.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Restates
/root/reference/pkg/src/aliasfft/dsfft.py:69-267 with layers as (depth, values,
active) tuples; classification and the aliased fallback reuse the exact / noisy
/ one-shot oracles.  Returns the entries dict and a layer trace comparable to
tests/golden/make_golden_dsfft.py's.
"""

from __future__ import annotations

import numpy as np

from . import oneshot as od
from .ffast import MULTI, SINGLE, bucket_values, classify_rows, exact_eps
from .rffast import search, thresholds, wrap  # noqa: F401  (wrap re-exported for tests)


def threshold(noise_std: float, floor: float, depth: int) -> float:
    return max(floor, 3.0 * noise_std / np.sqrt(1 << depth))


def initial(x, depth, thr):
    vals = bucket_values(x, 1 << depth, [0])[0]
    return depth, {i: complex(v) for i, v in enumerate(vals)}, {i for i, v in enumerate(vals)
                                                                if abs(v) > thr}


def expand(x, layer, thr):
    """expand_layer (dsfft.py:82-115)."""
    n = x.size
    pdepth, _, pactive = layer
    depth = pdepth + 1
    b = 1 << depth
    half = 1 << pdepth
    cands = sorted({c for i in pactive for c in (i, i + half)})
    if 2 * len(pactive) <= depth:
        sub = x[np.arange(b) * (n // b)]
        vals = {i: complex(np.dot(sub, np.exp(-2j * np.pi * i * np.arange(b) / b)) / b)
                for i in cands}
        computed = cands
    else:
        full = bucket_values(x, b, [0])[0]
        vals = {i: complex(v) for i, v in enumerate(full)}
        computed = list(vals)
    return depth, vals, {i for i in computed if abs(vals[i]) > thr}


def plan(n: int, seed: int):
    c = int(np.ceil(np.log2(n)))
    m = max(2, int(np.ceil(np.log2(n) ** (1.0 / 3.0))))
    anchors = [int(t) for t in np.random.default_rng(seed).integers(0, n, size=c)]
    t = np.arange(m - 1)
    weights = 1.5 * m / (m * m - 1.0) * (1.0 - 4.0 * ((2.0 * t - m + 2.0) / (2.0 * m)) ** 2)
    shifts = [anchors[j] + (1 << j) * r for j in range(c) for r in range(m)]
    return c, m, weights, shifts


def classify(x, layer, mode, seed, noise_std):
    """_classify_active (dsfft.py:118-174): (entries, multitons)."""
    n = x.size
    depth, _, active = layer
    b = 1 << depth
    act = sorted(active)
    entries, multi = {}, []
    if mode == "exact":
        vals = bucket_values(x, b, [0, 1, 2]).T
        eps = exact_eps(x)
        if act:
            st, f0 = classify_rows(vals[act], np.array(act), np.full(len(act), b), n, eps, eps)
            for g, i in enumerate(act):
                if st[g] == SINGLE:
                    entries[int(f0[g])] = complex(vals[i, 0])
                elif st[g] == MULTI:
                    multi.append(i)
        return entries, multi
    c, m, w, shifts = plan(n, seed)
    stacked = bucket_values(x, b, shifts).T
    energies = np.sum(np.abs(stacked) ** 2, axis=1)
    if noise_std > 0.0:
        base = noise_std / np.sqrt(b) * np.sqrt(len(shifts))
        floor = 1e-8 * np.sqrt(float(energies.max(initial=0.0)))
        t0, t1 = max(1.5 * base, floor), max(2.5 * base, floor)
    else:
        quiet = [i for i in range(b) if i not in active]
        t0, t1 = thresholds(energies[quiet] if quiet else energies, len(shifts), scale=energies)
    for i in act:
        y = stacked[i]
        if np.linalg.norm(y) <= t0:
            continue
        f, v, rn = search(y, i, b, n, c, m, w, shifts)
        if rn <= t1:
            entries[f] = v
        else:
            multi.append(i)
    return entries, multi


def resolve_aliased(x, b, buckets, k_remaining, a_m, seed):
    """dsfft.py:201-228 via the one-shot oracle on the chosen buckets."""
    n = x.size
    step = n // b
    p = max(12, int(np.ceil(a_m * np.log10(max(step, 10)))))
    rsh = od.random_shifts(n, p, seed)
    rows = od.measurement_rows(x, b, a_m, rsh)[buckets]
    counts = od.vote(rows, min(k_remaining, a_m * len(buckets)), a_m)
    out = {}
    for pos, bucket in enumerate(buckets):
        a = min(int(counts[pos]), a_m)
        if a == 0:
            continue
        cands = od.locate(rows[pos], a_m, a, "dt3", bucket, b, n)
        if cands is None:
            continue
        f, v = od.pursue(rows[pos, 3 * a_m:], rsh, cands, b, n)
        out.update(zip(f, v))
    return out


def calibrate(x, k):
    n = x.size
    b = min(n, 1 << max(0, int(np.ceil(np.log2(32 * k)))))
    vals = bucket_values(x, b, [0])[0]
    return float(np.sqrt(b * float(np.median(np.abs(vals) ** 2)) / np.log(2.0)))


def dsfft(x, k, mode="exact", seed=0, noise_std=0.0, theta=0.75, a_m=4, floor=1e-6):
    """dsfft (dsfft.py:244-267): returns (truncated, entries, trace)."""
    x = np.asarray(x, dtype=np.complex128)
    n = x.size
    max_depth = n.bit_length() - 1
    trace = []
    if mode != "exact" and noise_std <= 0.0:
        noise_std = calibrate(x, k)
    depth = min(max(0, int(np.ceil(np.log2(k)))), max_depth)
    layer = initial(x, depth, threshold(noise_std, floor, depth))
    while len(layer[2]) < theta * k and layer[0] < max_depth:
        layer = expand(x, layer, threshold(noise_std, floor, layer[0] + 1))
        trace.append(["expand", layer[0], len(layer[2])])
    entries, multi = classify(x, layer, mode, seed, noise_std)
    trace.append(["classify", layer[0], len(entries), len(multi)])
    while mode != "exact" and multi and layer[0] < max_depth:
        layer = expand(x, layer, threshold(noise_std, floor, layer[0] + 1))
        trace.append(["expand", layer[0], len(layer[2])])
        entries, multi = classify(x, layer, mode, seed, noise_std)
        trace.append(["classify", layer[0], len(entries), len(multi)])
    remaining = k - len(entries)
    if multi and remaining > 0:
        entries.update(resolve_aliased(x, 1 << layer[0], multi, remaining, a_m, seed))
    ranked = sorted(entries.items(), key=lambda kv: (-abs(kv[1]), kv[0]))
    return dict(ranked[:k]), entries, trace
