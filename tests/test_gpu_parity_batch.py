"""Config-sized parity against the reference, with an agreement report.

Goldens: tests/golden/batch_{c2,c3,c4dt3}.npz and golden_dsfft_c4_*db*.json, made by
running the reference itself (tests/golden/make_golden_batch.py, make_golden_dsfft.py)
on the BASELINE batch sizes — C2 all 64 signals, C3 16 seeds with the literal
511/512/513 plan and the reference's auto plan, C4-DT3 32 signals per SNR, C4-DSFFT
2 signals per SNR.  Inputs are regenerated on the host with generate_test_case
(bit-identical to the reference's) and decoded through the C ABI.

Bars (north_star), stated here and in the report:
  * exact sFFT-DT (C2, c128): vote counts identical; significant support
    {|v| > 1e-3} identical; values within 1e-9; zero-magnitude padding entries
    (ulp-chaotic on the reference itself) logged, not compared;
  * noisy sFFT-DT3 (C4, c64): as C2 with values within 1e-6 (the golden stores the
    c64-input values as complex64);
  * R-FFAST (C3): identical pre-truncation spectrum (positions and insertion order),
    rounds, unresolved; thresholds within 1e-12 rel; values within 1e-9 rel L2;
  * DSFFT (C4): identical layer trace and support, values within 1e-6;
  * every config: the GPU's L0/L1/L2 against the truth (signals.py:120-138) equals
    the reference's exactly (L0) and within 1e-6 * max(reference value, 1) (L1, L2).
A support mismatch is logged in the report with the entry magnitudes on either side
(a threshold-boundary case) before the assertion fails.

The report (L0/L1/L2 of GPU vs reference, of each vs truth, agreement counts and
every mismatch) is written to profiles/r02_parity.json when AFFT_PARITY_REPORT is
set (the committed report comes from such a run on a B200).
"""

from __future__ import annotations

import glob
import json
import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN_DIR, ROOT, cx

pytestmark = pytest.mark.gpu
SIG = 1e-3
REPORT: dict = {}


@pytest.fixture(scope="module", autouse=True)
def _write_report():
    yield
    if os.environ.get("AFFT_PARITY_REPORT") and REPORT:
        path = os.path.join(ROOT, "profiles", "r02_parity.json")
        old = {}
        if os.path.exists(path):
            with open(path) as fh:
                old = json.load(fh)
        old.update(REPORT)
        with open(path, "w") as fh:
            json.dump(old, fh, indent=1)


def _metrics(truth: dict, est: dict, tol: float = 0.1):
    """evaluate() of the reference (signals.py:120-138) on plain dicts."""
    keys = sorted(set(truth) | set(est))
    if not keys:
        return [0.0, 0.0, 0.0]
    mag = np.abs(np.array([truth.get(f, 0.0) - est.get(f, 0.0) for f in keys],
                          dtype=np.complex128))
    return [float(np.sum(mag > tol)), float(np.sum(mag)), float(np.sqrt(np.sum(mag ** 2)))]


def _truth(n, k, seed):
    from paper_2011_05749_b200.signals import draw_truth

    pos, coef = draw_truth(n, k, np.random.default_rng(seed))
    return {int(f): complex(c) for f, c in zip(pos, coef)}


def _summary(name, bar, rows, mismatches, extra=None):
    g_vs_r = np.array([r["gpu_vs_ref"] for r in rows])
    g_vs_t = np.array([r["gpu_vs_truth"] for r in rows])
    r_vs_t = np.array([r["ref_vs_truth"] for r in rows])
    rep = {
        "signals": len(rows), "bar": bar,
        "support_identical": int(sum(r["support_identical"] for r in rows)),
        "gpu_vs_ref": {"l0_max": float(g_vs_r[:, 0].max()), "l1_max": float(g_vs_r[:, 1].max()),
                       "l2_max": float(g_vs_r[:, 2].max())},
        "gpu_vs_truth_mean": {"l0": float(g_vs_t[:, 0].mean()), "l1": float(g_vs_t[:, 1].mean()),
                              "l2": float(g_vs_t[:, 2].mean())},
        "ref_vs_truth_mean": {"l0": float(r_vs_t[:, 0].mean()), "l1": float(r_vs_t[:, 1].mean()),
                              "l2": float(r_vs_t[:, 2].mean())},
        # L1 / L2 differences relative to max(reference value, 1): exactly recovered
        # signals have L1 ~ 1e-13 vs the truth, where only an absolute bar is meaningful
        "l_vs_truth_max_abs_diff": {
            "l0": float(np.abs(g_vs_t[:, 0] - r_vs_t[:, 0]).max()),
            "l1_rel": float((np.abs(g_vs_t[:, 1] - r_vs_t[:, 1]) / np.maximum(r_vs_t[:, 1], 1.0)).max()),
            "l2_rel": float((np.abs(g_vs_t[:, 2] - r_vs_t[:, 2]) / np.maximum(r_vs_t[:, 2], 1.0)).max()),
        },
        "mismatches": mismatches,
    }
    rep.update(extra or {})
    REPORT[name] = rep
    return rep


def _check_l_vs_truth(rep):
    d = rep["l_vs_truth_max_abs_diff"]
    assert d["l0"] == 0 and d["l1_rel"] <= 1e-6 and d["l2_rel"] <= 1e-6, d


def _mismatch(i, seed, got: dict, want: dict):
    only_g = sorted(set(got) - set(want))
    only_r = sorted(set(want) - set(got))
    return {"signal": i, "seed": int(seed),
            "only_gpu": [[int(f), abs(got[f])] for f in only_g[:20]],
            "only_ref": [[int(f), abs(want[f])] for f in only_r[:20]]}


# ----------------------------------------------------------------------------- sFFT-DT

TIE = 1e-9


def _dt_tie_margin(row, rsh, a, variant, bucket, b, n):
    """Smallest relative gap at a ranking decision of the reference's per-bucket solve
    (oneshot.py:161-257), replayed with the oracle on the bucket's measurements: the
    dt2 |P| ranking at the a-th candidate, and every pursuit prune step's |coef| ranking
    at the want-th atom.  A gap below TIE means the reference's own choice is decided
    by rounding (e.g. a bucket holding more unit-magnitude tones than its vote count:
    the merged least-squares fit recovers them all with |coef| = 1 +- ulp, and the
    prune keeps whichever rounding ranks first)."""
    from oracle import oneshot as od

    gaps = [np.inf]
    step = n // b
    if variant == "dt2":
        coeffs = od.lstsq_solution(od.hankel(row, 4, a),
                                   -np.array([row[4 + a + r] for r in range(a)]))
        cands = (bucket + b * np.arange(step)) % n
        pv = np.sort(np.abs(np.polyval(np.concatenate(([1.0 + 0j], coeffs[::-1])),
                                       od.unit_root(cands, n))))
        if a < step:
            gaps.append((pv[a] - pv[a - 1]) / max(pv[a], 1e-300))
    cands = od.locate(row, 4, a, variant, bucket, b, n)
    if not cands:
        return float(min(gaps))
    y = np.asarray(row[12:], dtype=np.complex128)
    shifts = np.asarray(rsh, dtype=np.int64)
    freqs = []
    for f in cands:
        for g in (f, (f + b) % n, (f - b) % n):
            if g not in freqs:
                freqs.append(g)
    atoms = od.unit_root(np.array(freqs)[None, :], n, shifts[:, None])
    want = min(len(cands), len(freqs), len(shifts))

    def fit(sup):
        coef = od.lstsq_solution(atoms[:, sup], y)
        return coef, float(np.linalg.norm(y - atoms[:, sup] @ coef))

    corr = np.sort(np.abs(atoms.conj().T @ y))[::-1]
    if want < corr.size:
        gaps.append((corr[want - 1] - corr[want]) / max(corr[want - 1], 1e-300))
    sup = np.argsort(-np.abs(atoms.conj().T @ y), kind="stable")[:want]
    coef, res = fit(sup)
    best = (sup, coef, res)
    for _ in range(od.SP_MAX_ITERS):
        if best[2] <= 1e-10 * max(1.0, float(np.linalg.norm(y))):
            break
        r = y - atoms[:, best[0]] @ best[1]
        fresh = np.argsort(-np.abs(atoms.conj().T @ r), kind="stable")[:want]
        merged = np.union1d(best[0], fresh)
        cm, _ = fit(merged)
        mags = np.sort(np.abs(cm))[::-1]
        if want < mags.size:
            gaps.append((mags[want - 1] - mags[want]) / max(mags[want - 1], 1e-300))
        pruned = np.sort(merged[np.argsort(-np.abs(cm), kind="stable")[:want]])
        coef, res = fit(pruned)
        if res >= best[2]:
            break
        best = (pruned, coef, res)
    return float(min(gaps))


def _classify_dt_mismatch(mm, n, k, snr, seed, b, p, variant, counts, c64):
    """Attach the tie margin of every bucket holding a mismatched entry; the mismatch
    is a logged boundary case iff every such bucket's margin is below TIE."""
    from oracle import oneshot as od
    from paper_2011_05749_b200.signals import generate_test_case

    x = generate_test_case(n, k, snr, seed).signal
    if c64:
        x = x.astype(np.complex64).astype(np.complex128)
    rsh = od.random_shifts(n, p, seed)
    rows = od.measurement_rows(x, b, 4, rsh)
    buckets = sorted({f % b for f, _ in mm["only_gpu"] + mm["only_ref"]})
    margins = {int(bk): _dt_tie_margin(rows[bk], rsh, int(counts[bk]), variant, int(bk), b, n)
               for bk in buckets}
    mm["bucket_tie_margin"] = margins
    mm["boundary_case"] = bool(mm.get("counts_identical", True)) and all(
        v < TIE for v in margins.values())
    return mm


def _dt_batch(name, tol):
    import _gen

    from paper_2011_05749_b200 import sfft_dt_batch

    d = np.load(os.path.join(GOLDEN_DIR, f"batch_{name}.npz"))
    meta = json.loads(str(d["meta"]))
    n, k, b, p, variant, c64 = (meta[key] for key in ("n", "k", "b", "p", "variant", "c64"))
    seeds = [int(s) for s in d["seed"]]
    snrs = ["exact" if s == 0 and name == "c2" else float(s) for s in d["snr"]]
    rows, mism, counts_ok = [], [], 0
    # one batched call per SNR group (C4: 32 signals per SNR; C2: all 64)
    groups = {}
    for i, s in enumerate(snrs):
        groups.setdefault(s, []).append(i)
    for snr, idx in groups.items():
        specs = [(n, k, snr, seeds[i], c64) for i in idx]
        xs = torch.stack([torch.from_numpy(x) for x in _gen.signals(
            specs, gb_per_worker=0.5 if n <= 1 << 22 else 2.0)]).cuda()
        res = sfft_dt_batch(xs, k, b, 4, p, variant, seeds=[seeds[i] for i in idx])
        del xs
        counts = res.counts.cpu().numpy()
        for j, i in enumerate(idx):
            want_counts = d["counts"][i].astype(np.int32)
            c_ok = bool(np.array_equal(counts[j], want_counts))
            counts_ok += c_ok
            a, z = int(d["off"][i]), int(d["off"][i + 1])
            want_all = {int(f): complex(v) for f, v in zip(d["pos"][a:z], d["val"][a:z])}
            want = {f: v for f, v in want_all.items() if abs(v) > SIG}
            got_all = res.full_spectrum(j).entries
            got = {f: v for f, v in got_all.items() if abs(v) > SIG}
            same = set(got) == set(want)
            vals_ok = same and all(abs(got[f] - v) <= tol for f, v in want.items())
            ta, tz = int(d["toff"][i]), int(d["toff"][i + 1])
            ref_tr = {int(f): want_all[int(f)] for f in d["trunc"][ta:tz]}
            gpu_tr = res.spectrum(j).entries
            truth = _truth(n, k, seeds[i])
            rows.append({"support_identical": same and vals_ok and c_ok,
                         "gpu_vs_ref": _metrics(ref_tr, gpu_tr),
                         "gpu_vs_truth": _metrics(truth, gpu_tr),
                         "ref_vs_truth": [float(v) for v in d["metrics"][i]]})
            if not (same and c_ok):
                m = _mismatch(i, seeds[i], got, want)
                m["counts_identical"] = c_ok
                if c_ok:
                    m = _classify_dt_mismatch(m, n, k, snr, seeds[i], b, p, variant,
                                              want_counts, c64)
                rows[-1]["boundary"] = m.get("boundary_case", False)
                mism.append(m)
    bar = ("vote counts identical; significant support {|v|>1e-3} identical; values within "
           f"{tol:g}; L0 vs truth identical, L1/L2 vs truth within 1e-6 max(L, 1) -- except "
           f"signals whose differing entries all sit in buckets where the reference's own "
           f"ranking decision (dt2 |P|, pursuit correlation or prune |coef|) has a relative "
           f"gap below {TIE:g}: logged as threshold-boundary cases")
    rep = _summary(name, bar, rows, mism, {"counts_identical": counts_ok})
    bad = [m for m in mism if not m.get("boundary_case")]
    assert not bad, bad[:3]
    _check_l_vs_truth(_summary(name + "_non_boundary", bar,
                               [r for r in rows if not r.get("boundary")] or rows, []))
    REPORT.pop(name + "_non_boundary", None)


def test_config2_all_64_signals():
    _dt_batch("c2", 1e-9)


def test_config4_dt3_32_per_snr():
    _dt_batch("c4dt3", 1e-6)


# ----------------------------------------------------------------------------- R-FFAST


def test_config3_16_seeds_both_plans():
    import _gen

    from paper_2011_05749_b200 import rffast_batch
    from paper_2011_05749_b200.peeling import SearchPlan, kay_weights

    d = np.load(os.path.join(GOLDEN_DIR, "batch_c3.npz"))
    meta = json.loads(str(d["meta"]))
    n, k, snr = meta["n"], meta["k"], meta["snr"]
    seeds = [int(s) for s in d["seed"]]
    limit = int(os.environ.get("AFFT_PARITY_C3_SEEDS", len(seeds)))
    seeds = seeds[:limit]
    rows = {"literal": [], "auto": []}
    mism = {"literal": [], "auto": []}
    specs = [(n, k, snr, s, False) for s in seeds]
    xd = torch.empty((len(seeds), n), dtype=torch.complex128, device="cuda")
    for i, x in enumerate(_gen.signals(specs, gb_per_worker=8.0)):
        xd[i].copy_(torch.from_numpy(x))
        del x
    for tag in ("literal", "auto"):
        m = meta[tag]
        plans = [SearchPlan(c=m["c"], m=m["m"], anchors=[int(a) for a in d[f"{tag}_anchors"][i]],
                            weights=kay_weights(m["m"])) for i in range(len(seeds))]
        assert all(f == m["factors"][0] for f in m["factors"])
        # one batched decode, every signal with its own search anchors
        res = rffast_batch(xd, k, m["factors"][0], plans)
        for i in range(len(seeds)):
            truth = _truth(n, k, seeds[i])
            a, z = int(d[f"{tag}_off"][i]), int(d[f"{tag}_off"][i + 1])
            want = {int(f): complex(v) for f, v in zip(d[f"{tag}_pos"][a:z], d[f"{tag}_val"][a:z])}
            got = res.full_spectrum(i).entries
            same = list(got) == list(want)
            if same and want:
                av = np.array([got[f] for f in want])
                bv = np.array(list(want.values()))
                same = bool(np.linalg.norm(av - bv) <= 1e-9 * np.linalg.norm(bv))
            t0, t1 = d[f"{tag}_thr"][i]
            rounds, unres = d[f"{tag}_ru"][i]
            same = (same and int(res.rounds[i]) == rounds and int(res.unresolved[i]) == unres
                    and abs(float(res.t0[i]) - t0) <= 1e-12 * t0
                    and abs(float(res.t1[i]) - t1) <= 1e-12 * t1)
            ta, tz = int(d[f"{tag}_toff"][i]), int(d[f"{tag}_toff"][i + 1])
            ref_tr = {int(f): want[int(f)] for f in d[f"{tag}_trunc"][ta:tz]}
            gpu_tr = res.spectrum(i).entries
            rows[tag].append({"support_identical": same, "gpu_vs_ref": _metrics(ref_tr, gpu_tr),
                              "gpu_vs_truth": _metrics(truth, gpu_tr),
                              "ref_vs_truth": [float(v) for v in d[f"{tag}_metrics"][i]]})
            if not same:
                mm = _mismatch(i, seeds[i], got, want)
                mm.update({"t0": [float(res.t0[i]), t0], "t1": [float(res.t1[i]), t1],
                           "rounds": [int(res.rounds[i]), int(rounds)]})
                mism[tag].append(mm)
        del res
    del xd
    bar = ("identical pre-truncation spectrum (order too), rounds, unresolved; thresholds within "
           "1e-12 rel; values within 1e-9 rel L2; L0 vs truth identical, L1/L2 within 1e-6 max(L, 1)")
    reps = [_summary(f"c3_{tag}", bar, rows[tag], mism[tag],
                     {"factors": meta[tag]["factors"][0]}) for tag in ("literal", "auto")]
    assert not mism["literal"] and not mism["auto"], (mism["literal"][:2], mism["auto"][:2])
    for rep in reps:
        _check_l_vs_truth(rep)


# ----------------------------------------------------------------------------- DSFFT


def test_config4_dsfft_per_snr():
    from paper_2011_05749_b200 import DsfftConfig, _device
    from paper_2011_05749_b200.dsfft import dsfft_device
    from conftest import dsfft_signal

    paths = sorted(glob.glob(os.path.join(GOLDEN_DIR, "golden_dsfft_c4_*db*.json")))
    assert paths
    rows, mism = [], []
    for path in paths:
        with open(path) as fh:
            case = json.load(fh)
        x = dsfft_signal(case)
        cfg = DsfftConfig(mode=case["mode"], seed=case["seed"], noise_std=case["noise_std"])
        trace = []
        entries = dsfft_device(_device.as_device_signal(x), case["k"], cfg, None, trace)
        ranked = sorted(entries.items(), key=lambda kv: (-abs(kv[1]), kv[0]))
        got = dict(ranked[: case["k"]])
        want = {f: cx(v) for f, v in case["truncated"]}
        same = trace == case["trace"] and set(got) == set(want) and all(
            abs(got[f] - v) <= 1e-6 for f, v in want.items())
        truth = _truth(case["n"], case["k"], case["seed"])
        ref_vs_truth = case.get("metrics") or _metrics(truth, want)
        rows.append({"support_identical": same, "gpu_vs_ref": _metrics(want, got),
                     "gpu_vs_truth": _metrics(truth, got), "ref_vs_truth": ref_vs_truth})
        if not same:
            mm = _mismatch(os.path.basename(path), case["seed"], got, want)
            mm["trace_identical"] = trace == case["trace"]
            mism.append(mm)
    bar = ("identical layer trace (depths, active counts, single/multi counts) and support; "
           "values within 1e-6; L0 vs truth identical, L1/L2 within 1e-6 max(L, 1)")
    rep = _summary("c4_dsfft", bar, rows, mism,
                   {"goldens": [os.path.basename(p) for p in paths]})
    assert not mism, mism[:3]
    _check_l_vs_truth(rep)
