"""Golden vectors for DSFFT, produced by running the REFERENCE (build container).

    python tests/golden/make_golden_dsfft.py            # small / medium cases
    python tests/golden/make_golden_dsfft.py --c4 20    # config 4 at one SNR (~8 min, ~40 GB)

Records the layer trace (depth, active count per expansion) by wrapping the
reference's expand_layer, the entries before truncation, and the output.  The
reference's small-matrix cap is lifted at runtime (MAX_DIM = 4096).
Config 4 follows the bench convention noise_std = sqrt(K * 10^(-snr/10))
(/root/reference/pkg/src/aliasfft/bench.py:142-148).
"""

from __future__ import annotations

import argparse
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
    ap = argparse.ArgumentParser()
    ap.add_argument("--c4", type=float, default=None)
    args = ap.parse_args()
    sys.dont_write_bytecode = True
    sys.path.insert(0, os.environ.get("ALIASFFT_REF", "/root/reference/pkg/src"))
    import aliasfft as ref  # noqa: E402

    sys.modules["aliasfft.smallnum"].MAX_DIM = 4096
    dmod = sys.modules["aliasfft.dsfft"]
    trace = []
    orig_expand = dmod.expand_layer
    orig_classify = dmod._classify_active

    def traced_expand(x, prev, ledger, thr):
        layer = orig_expand(x, prev, ledger, thr)
        trace.append(["expand", layer.depth, layer.m_d])
        return layer

    def traced_classify(x, layer, config, ledger):
        entries, multi = orig_classify(x, layer, config, ledger)
        trace.append(["classify", layer.depth, len(entries), len(multi)])
        return entries, multi

    dmod.expand_layer = traced_expand
    dmod._classify_active = traced_classify

    def run(n, k, snr, seed, mode, noise_std=0.0, positions=None, c64=False):
        trace.clear()
        case = ref.generate_test_case(n, k, snr, seed, positions=positions)
        x = case.signal
        if c64:
            x = x.astype(np.complex64).astype(np.complex128)
        cfg = ref.DsfftConfig(mode=mode, seed=seed, noise_std=noise_std)
        ledger = ref.SampleLedger(n)
        t = time.perf_counter()
        out = ref.dsfft(x, k, cfg, ledger)
        dt = time.perf_counter() - t
        return {"n": n, "k": k, "snr": snr, "seed": seed, "mode": mode, "noise_std": noise_std,
                "positions": positions, "c64": c64, "trace": list(trace),
                "truncated": [[int(f), cx(v)] for f, v in out.entries.items()],
                "truth": sorted(int(f) for f in case.truth.entries),
                "ledger": [ledger.count, ledger.unique_count], "ref_seconds": dt}

    if args.c4 is None:
        cases = [run(64, 5, "exact", 11, "exact", positions=[1, 6, 13, 20, 59])]
        for seed in range(3):
            cases.append(run(1 << 12, 4, "exact", seed, "exact"))
            cases.append(run(1 << 14, 16, "exact", seed, "exact"))
        for seed in range(2):
            cases.append(run(1 << 16, 16, 20.0, seed, "noisy",
                             noise_std=float(np.sqrt(16 * 10 ** (-2.0)))))
            cases.append(run(1 << 14, 8, 10.0, seed, "noisy"))  # calibrated noise_std
        n, k = 1 << 20, 256
        for snr in (10.0, 30.0):
            cases.append(run(n, k, snr, case_seed(n, k, snr, 0, 0), "noisy",
                             noise_std=float(np.sqrt(k * 10 ** (-snr / 10))), c64=True))
        # layer-count KAT of reference tests/test_dsfft.py:33-37 via the layer API
        case = ref.generate_test_case(64, 5, "exact", seed=11, positions=[1, 6, 13, 20, 59])
        layer = ref.initial_layer(case.signal, 0, None, 1e-6)
        counts = [layer.m_d]
        for _ in range(3):
            layer = orig_expand(case.signal, layer, None, 1e-6)
            counts.append(layer.m_d)
        out = {"generator": "tests/golden/make_golden_dsfft.py", "cases": cases,
               "layer_counts_n64": counts}
        path = os.path.join(HERE, "golden_dsfft.json")
    else:
        n, k, snr = 1 << 24, 4096, args.c4
        seed = case_seed(n, k, snr, 0, 0)
        out = run(n, k, snr, seed, "noisy", noise_std=float(np.sqrt(k * 10 ** (-snr / 10))),
                  c64=True)
        path = os.path.join(HERE, f"golden_dsfft_c4_{int(snr)}db.json")
    with open(path, "w") as fh:
        json.dump(out, fh, separators=(",", ":"))
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


if __name__ == "__main__":
    main()
