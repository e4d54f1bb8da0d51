"""Golden vectors for sFFT-DT1/2/3, produced by running the REFERENCE (build container).

    python tests/golden/make_golden_dt.py

Writes golden_dt.json: for each case the vote counts, the pre-truncation entries
(the dict sfft_dt builds, in insertion order), the truncated output and the
ledger.  Cases: small exact dt1/dt2/dt3, noisy dt3, BASELINE config 2
(N=2^22, K=1000, B=1024, p=15, dt2) and config 4's sFFT-DT3.0 leg (N=2^24,
K=4096, B=4096, p=15, complex64, 10/20/30 dB).
"""

from __future__ import annotations

import json
import os
import sys
import time
import zlib

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def cx(v):
    return [float(np.real(v)), float(np.imag(v))]


def case_seed(n, k, snr, seed_base, trial):
    tag = "exact" if snr == "exact" else f"{float(snr):.9g}"
    return zlib.crc32(f"{n}|{k}|{tag}|{seed_base}|{trial}".encode()) ^ (seed_base << 1)


def main():
    sys.dont_write_bytecode = True
    sys.path.insert(0, os.environ.get("ALIASFFT_REF", "/root/reference/pkg/src"))
    import aliasfft as ref  # noqa: E402
    from aliasfft.oneshot import (  # noqa: E402
        collect_moments, detect_sparsity, estimate_values, locate, truncate_spectrum,
    )

    def run(n, k, snr, b, p, variant, trial, c64=False):
        seed = case_seed(n, k, snr, 0, trial)
        case = ref.generate_test_case(n, k, snr, seed)
        x = case.signal
        if c64:
            x = x.astype(np.complex64).astype(np.complex128)
        cfg = ref.OneShotConfig(b=b, a_m=4, p=p, variant=variant, seed=seed)
        ledger = ref.SampleLedger(n)
        t = time.perf_counter()
        moments = collect_moments(x, cfg, ledger)
        counts = detect_sparsity(moments, k, cfg.a_m)
        entries = {}
        for pos, m in enumerate(moments):
            a = int(counts[pos])
            if a == 0:
                continue
            cands = locate(m, a, variant, b, n)
            if cands is None:
                continue
            sol = estimate_values(m, cands, b, n)
            for f, v in zip(sol.positions, sol.values):
                entries[f] = v
        trunc = truncate_spectrum(entries, n, k)
        dt = time.perf_counter() - t
        nz = np.flatnonzero(counts)
        return {"n": n, "k": k, "snr": snr, "seed": seed, "b": b, "p": p, "variant": variant,
                "c64": c64, "counts_nz": [[int(i), int(counts[i])] for i in nz],
                "entries": [[int(f), cx(v)] for f, v in entries.items()],
                "truncated": [[int(f), cx(v)] for f, v in trunc.entries.items()],
                "truth": sorted(int(f) for f in case.truth.entries),
                "ledger": [ledger.count, ledger.unique_count], "ref_seconds": dt}

    cases = []
    for variant in ("dt1", "dt2", "dt3"):
        for trial in range(3):
            cases.append(run(1 << 14, 16, "exact", 512, 12, variant, trial))
    for trial in range(2):
        cases.append(run(1 << 16, 16, 20.0, 2048, 12, "dt3", trial))
        cases.append(run(1 << 16, 16, 20.0, 2048, 12, "dt2", trial))
    for trial in range(3):
        cases.append(run(1 << 22, 1000, "exact", 1024, 15, "dt2", trial))
    for snr in (10.0, 20.0, 30.0):
        cases.append(run(1 << 24, 4096, snr, 4096, 15, "dt3", 0, c64=True))
    path = os.path.join(HERE, "golden_dt.json")
    with open(path, "w") as fh:
        json.dump({"generator": "tests/golden/make_golden_dt.py", "cases": cases}, fh,
                  separators=(",", ":"))
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


if __name__ == "__main__":
    main()
