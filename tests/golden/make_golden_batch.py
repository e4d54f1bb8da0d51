"""Config-sized golden batches, produced by running the REFERENCE (build container).

    python tests/golden/make_golden_batch.py c2            # 64 signals   (~1 min on 8 cores)
    python tests/golden/make_golden_batch.py c4dt3         # 32 per SNR   (~3 min)
    python tests/golden/make_golden_batch.py c3 [--seeds 16] [--workers 4]   (~8 min, ~8 GB/worker)
    python tests/golden/make_golden_batch.py c4dsfft --trials 1   # one more signal per SNR
                                                                  # (~8 min, ~40 GB each, serial)

Each run writes tests/golden/batch_<config>.npz.  Per signal: the seed (the
reference bench convention, bench.py:123-127, trial = signal index), the
pre-truncation entries in insertion order, the truncated support, the
reference's own L0/L1/L2 against the truth (signals.py:120-138) and — per
family — the vote counts (sFFT-DT), thresholds / rounds / unresolved (R-FFAST) or
the layer trace (DSFFT).  Calls are SURVEY Appendix A's; the reference's 64x64
small-matrix cap is lifted at runtime for C3/C4 (MAX_DIM = 4096), its
files untouched.  Values of complex64-input configs are stored as complex64
(their parity bar is 1e-6); everything else is stored exactly.
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
REF = os.environ.get("ALIASFFT_REF", "/root/reference/pkg/src")


def case_seed(n, k, snr, seed_base, trial):
    tag = "exact" if snr == "exact" else f"{float(snr):.9g}"
    return zlib.crc32(f"{n}|{k}|{tag}|{seed_base}|{trial}".encode()) ^ (seed_base << 1)


def _ref():
    sys.dont_write_bytecode = True
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import aliasfft as ref

    sys.modules["aliasfft.smallnum"].MAX_DIM = 4096
    return ref


def _metrics(ref, truth, est):
    m = ref.evaluate(truth, est)
    return [float(m.l0), float(m.l1), float(m.l2)]


# ----------------------------------------------------------------------------- sFFT-DT


def dt_one(job):
    n, k, snr, b, p, variant, trial, c64 = job
    ref = _ref()
    from aliasfft.oneshot import (
        collect_moments, detect_sparsity, estimate_values, locate, truncate_spectrum,
    )

    seed = case_seed(n, k, snr, 0, trial)
    case = ref.generate_test_case(n, k, snr, seed)
    x = case.signal
    if c64:
        x = x.astype(np.complex64).astype(np.complex128)
    cfg = ref.OneShotConfig(b=b, a_m=4, p=p, variant=variant, seed=seed)
    t = time.perf_counter()
    moments = collect_moments(x, cfg, None)
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
    return {"trial": trial, "seed": seed, "snr": snr, "counts": np.asarray(counts, np.int8),
            "pos": np.fromiter(entries.keys(), np.int64, len(entries)),
            "val": np.fromiter(entries.values(), np.complex128, len(entries)),
            "trunc": np.fromiter(trunc.entries.keys(), np.int64, len(trunc.entries)),
            "metrics": _metrics(ref, case.truth, trunc), "seconds": dt}


def save_dt(name, recs, meta, c64):
    recs = sorted(recs, key=lambda r: (float(r["snr"]) if r["snr"] != "exact" else 0.0,
                                       r["trial"]))
    off = np.cumsum([0] + [len(r["pos"]) for r in recs])
    toff = np.cumsum([0] + [len(r["trunc"]) for r in recs])
    val = np.concatenate([r["val"] for r in recs])
    np.savez_compressed(
        os.path.join(HERE, f"batch_{name}.npz"),
        meta=json.dumps(meta), trial=np.array([r["trial"] for r in recs]),
        seed=np.array([r["seed"] for r in recs], np.int64),
        snr=np.array([0.0 if r["snr"] == "exact" else float(r["snr"]) for r in recs]),
        counts=np.stack([r["counts"] for r in recs]),
        off=off, pos=np.concatenate([r["pos"] for r in recs]).astype(np.int32),
        val=val.astype(np.complex64) if c64 else val,
        toff=toff, trunc=np.concatenate([r["trunc"] for r in recs]).astype(np.int32),
        metrics=np.array([r["metrics"] for r in recs]),
        seconds=np.array([r["seconds"] for r in recs]))


# ----------------------------------------------------------------------------- R-FFAST


def rffast_one(job):
    n, k, snr, trial = job
    ref = _ref()
    from aliasfft.oneshot import truncate_spectrum
    from aliasfft.peeling import build_graph, noisy_thresholds, peel_decode

    seed = case_seed(n, k, snr, 0, trial)
    case = ref.generate_test_case(n, k, snr, seed)
    x = case.signal
    out = {"trial": trial, "seed": seed}
    plan_auto, sp_auto = ref.plan_cycles(n, k, "noisy", seed)
    for tag, factors in (("literal", [511, 512, 513]), ("auto", list(plan_auto.factors))):
        _, sp = ref.plan_cycles(n, k, "noisy", seed)
        t = time.perf_counter()
        graph = build_graph(x, ref.CyclePlan(factors, sp.shifts))
        sp.t0, sp.t1 = noisy_thresholds(graph)
        res = peel_decode(graph, "noisy", search_plan=sp, max_rounds=k + 4)
        trunc = truncate_spectrum(res.spectrum.entries, n, k)
        dt = time.perf_counter() - t
        ent = res.spectrum.entries
        out[tag] = {"factors": factors, "c": sp.c, "m": sp.m, "anchors": list(sp.anchors),
                    "t0": sp.t0, "t1": sp.t1, "rounds": res.rounds,
                    "unresolved": res.unresolved_multitons,
                    "pos": np.fromiter(ent.keys(), np.int64, len(ent)),
                    "val": np.fromiter(ent.values(), np.complex128, len(ent)),
                    "trunc": np.fromiter(trunc.entries.keys(), np.int64, len(trunc.entries)),
                    "metrics": _metrics(ref, case.truth, trunc), "seconds": dt}
        del graph
    return out


def save_rffast(recs):
    recs = sorted(recs, key=lambda r: r["trial"])
    arrays = {"trial": np.array([r["trial"] for r in recs]),
              "seed": np.array([r["seed"] for r in recs], np.int64)}
    meta = {"n": 511 * 512 * 513, "k": 1000, "snr": 20.0,
            "generator": "tests/golden/make_golden_batch.py c3"}
    for tag in ("literal", "auto"):
        rs = [r[tag] for r in recs]
        meta[tag] = {"factors": [r["factors"] for r in rs], "c": rs[0]["c"], "m": rs[0]["m"]}
        arrays[f"{tag}_anchors"] = np.array([r["anchors"] for r in rs], np.int64)
        arrays[f"{tag}_thr"] = np.array([[r["t0"], r["t1"]] for r in rs])
        arrays[f"{tag}_ru"] = np.array([[r["rounds"], r["unresolved"]] for r in rs], np.int64)
        arrays[f"{tag}_off"] = np.cumsum([0] + [len(r["pos"]) for r in rs])
        arrays[f"{tag}_pos"] = np.concatenate([r["pos"] for r in rs])
        arrays[f"{tag}_val"] = np.concatenate([r["val"] for r in rs])
        arrays[f"{tag}_toff"] = np.cumsum([0] + [len(r["trunc"]) for r in rs])
        arrays[f"{tag}_trunc"] = np.concatenate([r["trunc"] for r in rs])
        arrays[f"{tag}_metrics"] = np.array([r["metrics"] for r in rs])
        arrays[f"{tag}_seconds"] = np.array([r["seconds"] for r in rs])
    np.savez_compressed(os.path.join(HERE, "batch_c3.npz"), meta=json.dumps(meta), **arrays)


# ----------------------------------------------------------------------------- DSFFT


def dsfft_one(job):
    n, k, snr, trial = job
    ref = _ref()
    dmod = sys.modules["aliasfft.dsfft"]
    trace = []
    orig_expand, orig_classify = dmod.expand_layer, dmod._classify_active

    def traced_expand(x, prev, ledger, thr):
        layer = orig_expand(x, prev, ledger, thr)
        trace.append(["expand", layer.depth, layer.m_d])
        return layer

    def traced_classify(x, layer, config, ledger):
        entries, multi = orig_classify(x, layer, config, ledger)
        trace.append(["classify", layer.depth, len(entries), len(multi)])
        return entries, multi

    dmod.expand_layer, dmod._classify_active = traced_expand, traced_classify
    seed = case_seed(n, k, snr, 0, trial)
    case = ref.generate_test_case(n, k, snr, seed)
    x = case.signal.astype(np.complex64).astype(np.complex128)
    noise_std = float(np.sqrt(k * 10 ** (-snr / 10)))
    cfg = ref.DsfftConfig(mode="noisy", seed=seed, noise_std=noise_std)
    t = time.perf_counter()
    out = ref.dsfft(x, k, cfg, None)
    dt = time.perf_counter() - t
    return {"n": n, "k": k, "snr": snr, "seed": seed, "trial": trial, "mode": "noisy",
            "noise_std": noise_std, "positions": None, "c64": True, "trace": trace,
            "truncated": [[int(f), [float(v.real), float(v.imag)]] for f, v in out.entries.items()],
            "metrics": _metrics(ref, case.truth, out), "ref_seconds": dt}


# ----------------------------------------------------------------------------- main


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=["c2", "c4dt3", "c3", "c4dsfft"])
    ap.add_argument("--workers", type=int, default=os.cpu_count())
    ap.add_argument("--seeds", type=int, default=16)
    ap.add_argument("--trials", type=int, nargs="*", default=[1])
    args = ap.parse_args()
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    t0 = time.perf_counter()
    if args.config == "c2":
        jobs = [(1 << 22, 1000, "exact", 1024, 15, "dt2", t, False) for t in range(64)]
        with ctx.Pool(args.workers) as pool:
            recs = pool.map(dt_one, jobs, chunksize=1)
        save_dt("c2", recs, {"n": 1 << 22, "k": 1000, "b": 1024, "p": 15, "variant": "dt2",
                             "c64": False, "generator": "tests/golden/make_golden_batch.py c2"},
                False)
    elif args.config == "c4dt3":
        jobs = [(1 << 24, 4096, snr, 4096, 15, "dt3", t, True)
                for snr in (10.0, 20.0, 30.0) for t in range(32)]
        with ctx.Pool(args.workers) as pool:
            recs = pool.map(dt_one, jobs, chunksize=1)
        save_dt("c4dt3", recs, {"n": 1 << 24, "k": 4096, "b": 4096, "p": 15, "variant": "dt3",
                                "c64": True,
                                "generator": "tests/golden/make_golden_batch.py c4dt3"}, True)
    elif args.config == "c3":
        jobs = [(511 * 512 * 513, 1000, 20.0, t) for t in range(args.seeds)]
        with ctx.Pool(args.workers) as pool:
            recs = pool.map(rffast_one, jobs, chunksize=1)
        save_rffast(recs)
    else:
        for trial in args.trials:
            for snr in (10.0, 20.0, 30.0):
                rec = dsfft_one((1 << 24, 4096, snr, trial))
                path = os.path.join(HERE, f"golden_dsfft_c4_{int(snr)}db_t{trial}.json")
                with open(path, "w") as fh:
                    json.dump(rec, fh, separators=(",", ":"))
                print(f"wrote {path} ({rec['ref_seconds']:.0f} s)", flush=True)
    print(f"{args.config}: {time.perf_counter() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    main()
