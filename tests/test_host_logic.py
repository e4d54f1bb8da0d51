"""Host-side planning and bookkeeping (no GPU): the reference's KATs for them."""

import numpy as np
import pytest

from paper_2011_05749_b200 import (
    SampleLedger,
    SparseSpectrum,
    UnsupportedSizeError,
    evaluate,
    kay_weights,
    plan_cycles,
)
from paper_2011_05749_b200.bucketize import gather_indices, record_bucketization


class TestPlanning:  # reference tests/test_peeling.py:37-71
    def test_n20_uses_4_and_5(self):
        with pytest.warns(UserWarning):
            plan, _ = plan_cycles(20, 5, "exact")
        assert plan.factors == [4, 5] and plan.shifts == [0, 1, 2]

    def test_n504(self):
        assert plan_cycles(504, 6, "exact")[0].factors == [7, 8, 9]

    def test_rejections(self):
        for n in (31, 64):
            with pytest.raises(UnsupportedSizeError):
                plan_cycles(n, 2, "exact")

    def test_merging(self):
        assert plan_cycles(4095, 1, "exact")[0].factors == [5, 7, 9, 13]
        assert plan_cycles(4095, 8, "exact")[0].factors == [63, 65]

    def test_noisy_plan_shape(self):
        _, search = plan_cycles(4095, 4, "noisy", seed=9)
        assert (search.c, search.m) == (12, 3)
        assert search.shifts == [search.anchors[j] + (1 << j) * t
                                 for j in range(12) for t in range(3)]

    def test_config_plans(self):
        # the auto-planner does not pick the configs' factors
        with pytest.warns(UserWarning):
            assert plan_cycles(2097024, 256, "exact")[0].factors == [3, 43, 127, 128]
        assert plan_cycles(124950, 40, "exact")[0].factors == [294, 425]
        _, s = plan_cycles(511 * 512 * 513, 1000, "noisy", seed=0)
        assert (s.c, s.m) == (27, 3)


def test_kay_weights():
    assert np.allclose(kay_weights(3), [0.5, 0.5])
    for m in range(2, 65):
        assert abs(kay_weights(m).sum() - 1.0) < 1e-12
    with pytest.raises(ValueError):
        kay_weights(1)


def test_ledger_replay_matches_index_formula():
    n, b = 20, 4
    for tau in (0, 1, 5, -3, 19):
        ledger = SampleLedger(n)
        record_bucketization(ledger, n, b, [tau])
        assert ledger.touched == {(j * 5 - tau) % n for j in range(b)}
        assert ledger.count == b
    ledger = SampleLedger(124950)
    for b in (49, 50, 51):
        record_bucketization(ledger, 124950, b, [0, 1, 2])
    assert (ledger.count, ledger.unique_count) == (450, 444)
    assert list(gather_indices(24, 6, -2)) == [(j * 4 + 2) % 24 for j in range(6)]


def test_sparse_spectrum_and_evaluate():
    with pytest.raises(ValueError):
        SparseSpectrum(4, {4: 1.0})
    a = SparseSpectrum(8, {1: 1.0, 3: 1j})
    b = SparseSpectrum(8, {1: 1.0, 5: 0.05})
    m = evaluate(a, b)
    assert m.l0 == 1 and abs(m.l1 - 1.05) < 1e-12
    assert np.array_equal(a.to_dense()[[1, 3]], [1.0, 1j])


def test_seeded_shift_draws_are_the_reference_stream():
    """collect_moments' random shifts (oneshot.py:93-94) are kept per (n, p, seed): the
    kept value is numpy's own draw, a repeat is the same list, and the caller's copy is
    not the cached object."""
    from paper_2011_05749_b200.oneshot import OneShotConfig, random_shifts

    for n, p, seed in ((1 << 22, 15, 7), (4096, 12, 0), (1 << 24, 15, 123456789)):
        cfg = OneShotConfig(b=64, a_m=4, p=p, variant="dt3", seed=seed)
        want = [int(t) for t in np.random.default_rng(seed).choice(n, size=p, replace=False)]
        got = random_shifts(n, cfg)
        assert got == want
        got.append(-1)  # the caller may edit its list
        assert random_shifts(n, cfg) == want


def test_guided_parts_cover_the_batch_in_order():
    from paper_2011_05749_b200.dsfft import _guided_parts

    for count in (0, 1, 5, 32, 96, 97):
        for workers in (1, 3, 8):
            for cap in (1, 4, 8):
                parts = _guided_parts(list(range(count)), workers, cap)
                assert sum(parts, []) == list(range(count))
                sizes = [len(p) for p in parts]
                assert all(1 <= s <= cap for s in sizes)
                assert sizes == sorted(sizes, reverse=True)  # long chunks first
