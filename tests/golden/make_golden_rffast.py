"""Golden vectors for the R-FFAST path, produced by running the REFERENCE (build container).

    python tests/golden/make_golden_rffast.py [--c3]

Writes golden_rffast.json (single-tone searches, N=4095 and N=63*64*65 runs) and,
with --c3, golden_rffast_c3.json: BASELINE config 3 (N=511*512*513, K=1000,
20 dB) on one seeded signal, both the literal 511/512/513 plan with the
reference's own c=27/m=3 search plan and the reference's auto plan.  The
reference's 64x64 small-matrix cap is lifted at runtime
(aliasfft.smallnum.MAX_DIM = 4096); its files are untouched.
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
    ap.add_argument("--ref", default=os.environ.get("ALIASFFT_REF", "/root/reference/pkg/src"))
    ap.add_argument("--c3", action="store_true")
    args = ap.parse_args()
    sys.dont_write_bytecode = True
    sys.path.insert(0, args.ref)
    import aliasfft as ref  # noqa: E402
    from aliasfft.oneshot import truncate_spectrum  # noqa: E402
    from aliasfft.peeling import (  # noqa: E402
        BucketNode, SearchPlan, build_graph, noisy_thresholds, peel_decode, singleton_search_noisy,
    )

    sys.modules["aliasfft.smallnum"].MAX_DIM = 4096

    def run(n, k, snr, seed, factors=None, search=None, snr_hint=None):
        case = ref.generate_test_case(n, k, snr, seed)
        x = case.signal
        plan_auto, search_auto = ref.plan_cycles(n, k, "noisy", seed)
        if search is None:
            search = search_auto
            if snr_hint is not None and snr_hint < 5.0:
                search = SearchPlan(c=search.c, m=search.m + 1, anchors=search.anchors,
                                    weights=ref.kay_weights(search.m + 1))
        factors = factors or plan_auto.factors
        ledger = ref.SampleLedger(n)
        t = time.perf_counter()
        graph = build_graph(x, ref.CyclePlan(list(factors), search.shifts), ledger)
        search.t0, search.t1 = noisy_thresholds(graph)
        res = peel_decode(graph, "noisy", search_plan=search, max_rounds=k + 4)
        trunc = truncate_spectrum(res.spectrum.entries, n, k)
        dt = time.perf_counter() - t
        return {
            "n": n, "k": k, "snr": snr, "seed": seed, "factors": list(factors),
            "c": search.c, "m": search.m, "anchors": list(search.anchors),
            "t0": search.t0, "t1": search.t1, "rounds": res.rounds,
            "unresolved": res.unresolved_multitons,
            "recovered": [[int(f), cx(v)] for f, v in res.spectrum.entries.items()],
            "truncated": [[int(f), cx(v)] for f, v in trunc.entries.items()],
            "truth": sorted(int(f) for f in case.truth.entries),
            "ledger": [ledger.count, ledger.unique_count], "ref_seconds": dt,
        }

    if not args.c3:
        out = {"generator": "tests/golden/make_golden_rffast.py"}
        # singleton searches (reference tests/test_peeling.py:174-206 shapes)
        searches = []
        n = 4095
        _, sp = ref.plan_cycles(n, 2, "noisy", seed=4)
        for f in (17, 2000, 4094):
            x = ref.inverse_dft(ref.SparseSpectrum(n, {f: np.exp(0.9j)}))
            g = build_graph(x, ref.CyclePlan([63], sp.shifts))
            node = g.cycles[0][f % 63]
            f0, v, rn = singleton_search_noisy(node, sp, 63, n)
            searches.append({"n": n, "b": 63, "c": sp.c, "m": sp.m, "anchors": sp.anchors,
                             "residual": [cx(z) for z in node.residual], "index": node.index,
                             "f0": f0, "value": cx(v), "resnorm": rn})
        for seed in range(24):
            n, b = 512, 16
            rng = np.random.default_rng(seed)
            f = int(rng.integers(0, n))
            case = ref.generate_test_case(n, 1, 0.0, seed=seed, positions=[f])
            anchors = [int(t) for t in rng.integers(0, n, size=9)]
            sp = SearchPlan(c=9, m=3, anchors=anchors, weights=ref.kay_weights(3))
            g = build_graph(case.signal, ref.CyclePlan([b], sp.shifts))
            node = g.cycles[0][f % b]
            f0, v, rn = singleton_search_noisy(node, sp, b, n)
            searches.append({"n": n, "b": b, "c": 9, "m": 3, "anchors": anchors,
                             "residual": [cx(z) for z in node.residual], "index": node.index,
                             "f0": f0, "value": cx(v), "resnorm": rn, "truth": f})
        out["searches"] = searches
        runs = []
        for seed in range(4):
            runs.append(run(4095, 4, 10.0, seed))
        runs.append(run(4095, 4, 3.0, 7, snr_hint=3.0))
        for seed in range(2):
            runs.append(run(63 * 64 * 65, 20, 20.0, seed))
        out["runs"] = runs
        path = os.path.join(HERE, "golden_rffast.json")
    else:
        n, k = 511 * 512 * 513, 1000
        seed = case_seed(n, k, 20.0, 0, 0)
        _, sp = ref.plan_cycles(n, k, "noisy", seed)
        out = {"generator": "tests/golden/make_golden_rffast.py --c3",
               "literal": run(n, k, 20.0, seed, factors=[511, 512, 513], search=sp),
               "auto": run(n, k, 20.0, seed)}
        path = os.path.join(HERE, "golden_rffast_c3.json")
    with open(path, "w") as fh:
        json.dump(out, fh, separators=(",", ":"))
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


if __name__ == "__main__":
    main()
