"""GPU FFAST (exact peeling) parity against the reference goldens and the oracle.

Parity bar (BASELINE.json north_star): the pre-truncation support
is bit-exact and in the reference's insertion order; values within 1e-9
relative L2 (complex128 inputs) or 1e-4 (complex64 inputs, where the reference
ran on the exact upcast); rounds and unresolved multi-ton counts identical.
The truncated output is compared too, with the documented exception of
|v| ties at the k-th rank.
"""

import os
import numpy as np
import pytest
import torch

from conftest import case_seed, cx, golden_signal
from oracle import ffast as of

pytestmark = pytest.mark.gpu


def _rel_l2(got: dict, want: dict) -> float:
    keys = list(want)
    a = np.array([got[f] for f in keys])
    b = np.array([want[f] for f in keys])
    return float(np.linalg.norm(a - b) / max(1e-300, np.linalg.norm(b)))


def _check_case(case, res, i):
    full = res.full_spectrum(i).entries
    want = {f: cx(v) for f, v in case["recovered"]}
    assert list(full) == list(want), "support / insertion order differs"
    tol = 1e-4 if case["c64"] else 1e-9
    if want:
        assert _rel_l2(full, want) <= tol
    assert int(res.rounds[i]) == case["rounds"]
    assert int(res.unresolved[i]) == case["unresolved"]
    trunc = set(res.spectrum(i).entries)
    want_t = {f for f, _ in case["truncated"]}
    if trunc != want_t:  # only a |v| tie at the k-th rank may change the kept set
        mags = sorted((abs(cx(v)) for _, v in case["recovered"]), reverse=True)
        k = case["k"]
        assert len(mags) > k and abs(mags[k - 1] - mags[k]) < 1e-6, (trunc, want_t)


def test_goldens_one_call_per_case(golden_ffast):
    from paper_2011_05749_b200 import ffast_batch

    for case in golden_ffast["ffast"]:
        x = golden_signal(case)
        res = ffast_batch(x[None, :], case["k"], case["factors"])
        _check_case(case, res, 0)


def test_goldens_batched(golden_ffast):
    """Config 1 and config 5 cases as one batch each (the throughput path)."""
    from paper_2011_05749_b200 import ffast_batch

    for n in (124950, 2097024):
        cases = [c for c in golden_ffast["ffast"] if c["n"] == n]
        xs = np.stack([golden_signal(c) for c in cases])
        res = ffast_batch(torch.from_numpy(xs).cuda(), cases[0]["k"], cases[0]["factors"])
        for i, case in enumerate(cases):
            _check_case(case, res, i)


def test_drop_in_ffast_api(golden_ffast):
    from paper_2011_05749_b200 import CyclePlan, SampleLedger, ffast

    for case in golden_ffast["ffast"][:12]:
        x = golden_signal(case)
        ledger = SampleLedger(case["n"])
        out = ffast(x, case["k"], ledger, plan=CyclePlan(case["factors"], [0, 1, 2]))
        assert set(out.entries) == {f for f, _ in case["truncated"]}
        assert [ledger.count, ledger.unique_count] == case["ledger"]


def test_graph_api_census_and_states(golden_ffast):
    """build_graph + classify_exact + peel_decode: N=20 KAT and node states vs reference."""
    from paper_2011_05749_b200 import CyclePlan, NodeState, evaluate, generate_test_case, peel_decode
    from paper_2011_05749_b200.peeling import build_graph, classify_exact, exact_thresholds

    case = generate_test_case(20, 5, "exact", seed=7, positions=[1, 3, 5, 10, 13])
    plan = CyclePlan([4, 5], [0, 1, 2])
    graph = build_graph(case.signal, plan)
    eps = exact_thresholds(case.signal)
    census = {}
    for nodes, b in zip(graph.cycles, graph.factors):
        for node in nodes:
            census[(b, node.index)] = classify_exact(node, eps, eps, b, 20)
    assert [census[k].value for k in sorted(census)] == [
        "zero-ton", "multi-ton", "single-ton", "single-ton",
        "multi-ton", "single-ton", "zero-ton", "multi-ton", "zero-ton"]
    fresh = build_graph(case.signal, plan)
    res = peel_decode(fresh, "exact", eps_zero=eps, eps_ratio=eps, max_rounds=9)
    assert evaluate(case.truth, res.spectrum).l2 < 1e-9
    assert res.unresolved_multitons == 0 and res.rounds <= 4
    # conservation: every residual equals vec minus the recovered tones of its residue
    shifts = np.array(plan.shifts)
    for nodes, b in zip(fresh.cycles, fresh.factors):
        for node in nodes:
            exp = node.vec.copy()
            for f, v in fresh.recovered.items():
                if f % b == node.index:
                    exp -= v * np.exp(-2j * np.pi * (shifts * f % 20) / 20)
            assert np.linalg.norm(node.residual - exp) < 1e-8
    # node states after decode match the reference's, for every golden that stored them
    for gc in golden_ffast["ffast"]:
        if gc["states"] is None or gc["n"] > 5000:
            continue
        x = golden_signal(gc)
        g = build_graph(x, CyclePlan(gc["factors"], [0, 1, 2]))
        e = exact_thresholds(x)
        peel_decode(g, "exact", eps_zero=e, eps_ratio=e, max_rounds=gc["k"] + 4)
        assert [nd.state.value for cyc in g.cycles for nd in cyc] == gc["states"]


def test_edge_cases():
    from paper_2011_05749_b200 import NodeState, ffast, inverse_dft, peel_decode, plan_cycles
    from paper_2011_05749_b200 import SparseSpectrum, CyclePlan
    from paper_2011_05749_b200.peeling import BucketNode, build_graph, exact_thresholds, subtract

    # zero signal: empty in one round, every node ZERO_TON (reference test_peeling.py:265-273)
    plan, _ = plan_cycles(504, 3, "exact")
    graph = build_graph(np.zeros(504, dtype=complex), plan)
    r = peel_decode(graph, "exact", eps_zero=1e-12, eps_ratio=1e-12, max_rounds=7)
    assert r.spectrum.entries == {} and r.rounds == 1
    assert all(nd.state is NodeState.ZERO_TON for cyc in graph.cycles for nd in cyc)
    # saturated graph: nothing peels, 9 unresolved (test_peeling.py:275-287)
    x = inverse_dft(SparseSpectrum(20, {f: np.exp(0.1j * f) for f in range(10)}))
    with pytest.warns(UserWarning):
        plan, _ = plan_cycles(20, 10, "exact")
    g = build_graph(x, plan)
    e = exact_thresholds(x)
    r = peel_decode(g, "exact", eps_zero=e, eps_ratio=e, max_rounds=14)
    assert r.spectrum.entries == {} and r.unresolved_multitons == 9 and r.rounds == 1
    # k = 0 and subtract semantics
    assert ffast(np.zeros(20, dtype=complex), 0).entries == {}
    node = BucketNode(0, 2, np.ones(3, dtype=complex))
    with pytest.raises(ValueError):
        subtract(node, 5, 1.0, [0, 1, 2], 20, 4)
    subtract(node, 6, 0.0, [0, 1, 2], 20, 4)
    assert np.allclose(node.residual, node.vec)
    # soundness against the dense oracle (test_peeling.py:315-322)
    from paper_2011_05749_b200 import dense_dft, generate_test_case

    for seed in range(10):
        case = generate_test_case(504, 6, "exact", seed=seed)
        out = ffast(case.signal, 6)
        dense = dense_dft(case.signal)
        assert set(out.entries) <= set(case.truth.entries)
        for f, v in out.entries.items():
            assert abs(v - dense[f]) < 1e-6


def test_config5_full_batch_vs_oracle():
    """Config 5 shape (N=2,097,024, K=256, 127/128/129, complex64) on a 256-signal batch:
    the pre-truncation support of EVERY signal equals the oracle's bit for bit, in
    insertion order (the reference itself emits occasional spurious singletons, so
    "recovered is a subset of truth" is not a valid property), and >= 99% of all
    recovered tones are true tones within 1e-4."""
    from paper_2011_05749_b200 import ffast_batch
    from paper_2011_05749_b200.signals import draw_truth

    n, k, factors, batch = 2097024, 256, [127, 128, 129], 256
    dev = torch.device("cuda")
    spec = torch.zeros((batch, n), dtype=torch.complex128, device=dev)
    truths = []
    for i in range(batch):
        pos, coef = draw_truth(n, k, np.random.default_rng(case_seed(n, k, "exact", 0, i)))
        truths.append(dict(zip(pos.tolist(), coef.tolist())))
        spec[i, torch.from_numpy(pos).to(dev)] = torch.from_numpy(coef).to(dev)
    x = (torch.fft.ifft(spec, dim=1) * n).to(torch.complex64)
    del spec
    res = ffast_batch(x, k, factors)
    xh = x.cpu().numpy()
    good = total = 0
    for i in range(batch):
        got = res.full_spectrum(i).entries
        _, o = of.ffast(xh[i].astype(np.complex128), k, factors)
        assert list(o["recovered"]) == list(got), i
        assert int(res.rounds[i]) == o["rounds"] and int(res.unresolved[i]) == o["unresolved"]
        for f, v in got.items():
            total += 1
            good += f in truths[i] and abs(v - truths[i][f]) < 1e-4
    assert good >= 0.99 * total


def test_bench_synthesis_matches_generate_test_case():
    """bench.py synthesises config 5 on the device (numpy truth draws, cuFFT inverse,
    complex64); the signals must be the reference generator's (signals.py:81-117) for
    the same case seeds, up to complex64 rounding."""
    import sys

    from paper_2011_05749_b200 import generate_test_case

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import bench

    dev = torch.device("cuda")
    x, truths = bench.synth_batch(bench.N_SIG, bench.K, "exact", [5, 6], torch.complex64, dev)
    for i in range(2):
        seed = bench.case_seed(bench.N_SIG, bench.K, "exact", 0, 5 + i)
        case = generate_test_case(bench.N_SIG, bench.K, "exact", seed=seed)
        assert sorted(case.truth.entries) == truths[i].tolist()
        want = case.signal.astype(np.complex64)
        got = x[i].cpu().numpy()
        assert np.max(np.abs(got - want)) <= 1e-5 * np.max(np.abs(want))


def test_tree_walk_decoder(golden_ffast):
    """The paper's Fig. 5 tree-walk decoder (peel_decode(..., decoder="tree"),
    afft_peel_tree_exact; a non-goal of the reference, "identical output to
    Fig. 4 with fewer identifications"): on every reference golden, the recovered set is
    the reference's pre-truncation spectrum (values within the golden's tolerance, same
    unresolved count), and the identifications are fewer than the reference's round
    decoder performs (every live node, every round: at least nodes x rounds / 2 here)."""
    from paper_2011_05749_b200 import CyclePlan, peel_decode
    from paper_2011_05749_b200.peeling import build_graph, exact_thresholds

    for case in golden_ffast["ffast"]:
        x = golden_signal(case)
        g_tree = build_graph(x, CyclePlan(case["factors"], [0, 1, 2]))
        g_round = build_graph(x, CyclePlan(case["factors"], [0, 1, 2]))
        eps = exact_thresholds(x)
        tree = peel_decode(g_tree, "exact", eps, eps, max_rounds=case["k"] + 4, decoder="tree")
        rnd = peel_decode(g_round, "exact", eps, eps, max_rounds=case["k"] + 4)
        want = {f: cx(v) for f, v in case["recovered"]}
        got = tree.spectrum.entries
        if case["c64"]:
            # complex64 inputs: the rounding floor sits near the thresholds, so a
            # subtraction order other than the reference's may drop or add a tone that is
            # not in the signal (config 5 seed 21's 257th tone); the true tones agree
            truth = {int(f) for f in case["truth"]}
            assert set(got) & truth == set(want) & truth
            assert len(set(got) ^ set(want)) <= 1
            common = {f: want[f] for f in set(got) & set(want)}
            assert _rel_l2(got, common) <= 1e-4
        else:
            assert set(got) == set(want)
            assert set(got) == set(rnd.spectrum.entries)
            if want:
                assert _rel_l2(got, want) <= 1e-9
            assert tree.unresolved_multitons == case["unresolved"]
        nodes = sum(case["factors"])
        assert tree.identifications is not None and tree.identifications >= nodes // 2
        assert tree.identifications < nodes * case["rounds"] or case["rounds"] <= 1
