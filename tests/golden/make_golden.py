"""Generate golden vectors by running the REFERENCE implementation (build container only).

    python tests/golden/make_golden.py [--ref /root/reference/pkg/src]

Imports the read-only reference package, runs it on seeded inputs for the
hot-path functions, and writes JSON fixtures next to this script.  Floats are
stored with repr() so they round-trip exactly; complex values as [re, im].
The fixtures travel with the repo; the reference does not (it is absent on the
GPU box), so tests read only these files.  Re-run after changing what is
captured; the script is deterministic.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import zlib

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def cx(v) -> list:
    return [float(np.real(v)), float(np.imag(v))]


def case_seed(n, k, snr, seed_base, trial):
    """bench._case_seed (/root/reference/pkg/src/aliasfft/bench.py:123-127)."""
    tag = "exact" if snr == "exact" else f"{float(snr):.9g}"
    return zlib.crc32(f"{n}|{k}|{tag}|{seed_base}|{trial}".encode()) ^ (seed_base << 1)


def signal_digest(x: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(x, dtype=np.complex128).tobytes()).hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default=os.environ.get("ALIASFFT_REF", "/root/reference/pkg/src"))
    args = ap.parse_args()
    sys.dont_write_bytecode = True
    sys.path.insert(0, args.ref)
    import aliasfft as ref  # noqa: E402
    from aliasfft.bucketize import bucketize  # noqa: E402
    from aliasfft.oneshot import truncate_spectrum  # noqa: E402
    from aliasfft.peeling import build_graph, exact_thresholds, peel_decode  # noqa: E402

    out = {"generator": "tests/golden/make_golden.py", "reference": "aliasfft 0.1.0"}

    # 1. generate_test_case digests: pins the input model bit for bit
    gens = []
    for n, k, snr, seed in [(20, 5, "exact", 7), (64, 5, "exact", 11), (504, 6, "exact", 3),
                            (4095, 4, 10.0, 0), (4095, 4, 15.0, 5), (124950, 40, "exact", None),
                            (2097024, 256, "exact", None), (1 << 16, 16, 20.0, 2)]:
        if seed is None:
            seed = case_seed(n, k, snr, 0, 0)
        x = ref.generate_test_case(n, k, snr, seed).signal
        gens.append({"n": n, "k": k, "snr": snr, "seed": seed, "sha256": signal_digest(x),
                     "x0": cx(x[0]), "xlast": cx(x[-1])})
    out["generate_test_case"] = gens

    # 2. bucketize: exhaustive small alias sums and config-shaped stages
    rng = np.random.default_rng(2024)
    buck = []
    for n in (8, 12, 20, 24):
        x = rng.normal(size=n) + 1j * rng.normal(size=n)
        for b in [d for d in range(1, n + 1) if n % d == 0]:
            for tau in (-3, 0, 1, 2, 5, n - 1, n + 4):
                vals = bucketize(x, b, tau).values
                buck.append({"x": [cx(v) for v in x], "b": b, "tau": tau,
                             "values": [cx(v) for v in vals]})
    for n, k, factors, shifts, c64 in [
        (124950, 40, [49, 50, 51], [0, 1, 2], False),
        (2097024, 256, [127, 128, 129], [0, 1, 2], True),
        (1 << 22, 1000, [1024], list(range(-4, 8)), False),
        (511 * 512 * 8, 8, [511, 512], [0, 1, 2, 7, 1000, -5], False),
    ]:
        seed = case_seed(n, k, "exact", 0, 0)
        x = ref.generate_test_case(n, k, "exact", seed).signal
        if c64:
            x = x.astype(np.complex64).astype(np.complex128)
        for b in factors:
            for tau in shifts:
                vals = bucketize(x, b, tau).values
                buck.append({"gen": {"n": n, "k": k, "snr": "exact", "seed": seed, "c64": c64},
                             "b": b, "tau": tau, "values": [cx(v) for v in vals]})
    out["bucketize"] = buck

    # 3. FFAST with explicit plans (configs 1 and 5 of BASELINE.json + small KAT sizes)
    ff = []

    def run_ffast(n, k, factors, seed, c64=False, positions=None, snr="exact"):
        case = ref.generate_test_case(n, k, snr, seed, positions=positions)
        x = case.signal
        if c64:
            x = x.astype(np.complex64).astype(np.complex128)
        ledger = ref.SampleLedger(n)
        graph = build_graph(x, ref.CyclePlan(list(factors), [0, 1, 2]), ledger)
        eps = exact_thresholds(x)
        res = peel_decode(graph, "exact", eps_zero=eps, eps_ratio=eps, max_rounds=k + 4)
        trunc = truncate_spectrum(res.spectrum.entries, n, k)
        states = [node.state.value for cyc in graph.cycles for node in cyc]
        ff.append({
            "n": n, "k": k, "factors": list(factors), "seed": seed, "c64": c64,
            "positions": None if positions is None else list(positions), "snr": snr,
            "eps": eps, "rounds": res.rounds, "unresolved": res.unresolved_multitons,
            "recovered": [[int(f), cx(v)] for f, v in res.spectrum.entries.items()],
            "truncated": [[int(f), cx(v)] for f, v in trunc.entries.items()],
            "truth": sorted(int(f) for f in case.truth.entries),
            "ledger": [ledger.count, ledger.unique_count],
            "states": states if len(states) <= 600 else None,
        })

    run_ffast(20, 5, [4, 5], 7, positions=[1, 3, 5, 10, 13])
    for seed in range(6):
        run_ffast(504, 6, [7, 8, 9], seed)
    for seed in range(4):
        run_ffast(4095, 8, [63, 65], seed)
    for trial in range(10):
        run_ffast(124950, 40, [49, 50, 51], case_seed(124950, 40, "exact", 0, trial))
    for trial in range(6):
        run_ffast(2097024, 256, [127, 128, 129], case_seed(2097024, 256, "exact", 0, trial),
                  c64=True)
    out["ffast"] = ff

    path = os.path.join(HERE, "golden_ffast.json")
    with open(path, "w") as fh:
        json.dump(out, fh, separators=(",", ":"))
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


if __name__ == "__main__":
    main()
