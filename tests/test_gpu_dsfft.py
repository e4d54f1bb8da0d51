"""GPU DSFFT parity against the reference goldens (config 4's DSFFT leg included when its
golden exists).  Bar: identical layer trace (depths, active counts, single/multi counts
per classification), identical output support, values within 1e-9 (complex128) /
1e-6 (complex64), identical sample ledger."""

import glob
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN_DIR, cx, dsfft_signal

pytestmark = pytest.mark.gpu


def _check(case, trace, out, ledger=None):
    assert trace == case["trace"]
    want = {f: cx(v) for f, v in case["truncated"]}
    assert set(out.entries) == set(want), sorted(set(out.entries) ^ set(want))[:10]
    tol = 1e-6 if case["c64"] else 1e-9
    for f, v in want.items():
        assert abs(out.entries[f] - v) <= tol
    if ledger is not None:
        assert [ledger.count, ledger.unique_count] == case["ledger"]


def _run(case, with_ledger=True):
    from paper_2011_05749_b200 import DsfftConfig, SampleLedger, SparseSpectrum, _device
    from paper_2011_05749_b200.dsfft import dsfft_device

    x = dsfft_signal(case)
    cfg = DsfftConfig(mode=case["mode"], seed=case["seed"], noise_std=case["noise_std"])
    ledger = SampleLedger(case["n"]) if with_ledger else None
    trace = []
    entries = dsfft_device(_device.as_device_signal(x), case["k"], cfg, ledger, trace)
    ranked = sorted(entries.items(), key=lambda kv: (-abs(kv[1]), kv[0]))
    return trace, SparseSpectrum(case["n"], dict(ranked[: case["k"]])), ledger


def test_dsfft_goldens(golden_dsfft):
    for case in golden_dsfft["cases"]:
        trace, out, ledger = _run(case)
        _check(case, trace, out, ledger)


def test_layer_api_kat(golden_dsfft):
    from paper_2011_05749_b200 import dsfft, evaluate, expand_layer, generate_test_case, initial_layer

    case = generate_test_case(64, 5, "exact", seed=11, positions=[1, 6, 13, 20, 59])
    layer = initial_layer(case.signal, 0, None, 1e-6)
    counts = [layer.m_d]
    for _ in range(3):
        layer = expand_layer(case.signal, layer, None, 1e-6)
        counts.append(layer.m_d)
    assert counts == [1, 2, 4, 5]
    assert evaluate(case.truth, dsfft(case.signal, 5)).l2 < 1e-9
    # parent = sum of children (reference tests/test_dsfft.py:39-48)
    x = generate_test_case(128, 6, "exact", seed=3).signal
    parent = initial_layer(x, 3, None, 1e-6)
    child = initial_layer(x, 4, None, 1e-6)
    for i in range(parent.b):
        assert abs(parent.values[i] - (child.values[i] + child.values[i + parent.b])) < 1e-9


def test_dsfft_errors_and_probabilities():
    from paper_2011_05749_b200 import (UnsupportedSizeError, dsfft, non_aliasing_probability,
                                       non_aliasing_probability_limit)

    with pytest.raises(UnsupportedSizeError):
        dsfft(np.zeros(100, complex), 3)
    assert dsfft(np.zeros(64, complex), 0).entries == {}
    assert abs(non_aliasing_probability_limit(4, 8) - 0.4101) < 5e-3
    assert abs(non_aliasing_probability(64 * 8, 4, 8) - 0.4101) < 2e-2


C4 = sorted(glob.glob(os.path.join(GOLDEN_DIR, "golden_dsfft_c4_*db.json")))


@pytest.mark.parametrize("path", C4, ids=[os.path.basename(p) for p in C4])
def test_config4_dsfft_vs_reference(path):
    """BASELINE config 4, DSFFT leg: N=2^24, K=4096, complex64, noisy (one seeded signal)."""
    with open(path) as fh:
        case = json.load(fh)
    trace, out, _ = _run(case, with_ledger=False)
    _check(case, trace, out)


def test_dsfft_goldens_active_fallback(golden_dsfft, monkeypatch):
    """Deep full layers take their active set in one pass over the resident spectrum
    with a one-CTA sort (dsfft.cu: alias_active); above the sort's capacity the loop
    falls back to values + count / scan / write.  Forcing a capacity of 1 routes every
    deep layer through the fallback: the goldens must not change."""
    monkeypatch.setenv("AFFT_ACTIVE_SORT_CAP", "1")
    for case in golden_dsfft["cases"]:
        trace, out, ledger = _run(case)
        _check(case, trace, out, ledger)


def _entries_lazy_and_full(case, monkeypatch, probe0=None):
    """The native loop's entries dict with probe classifies (no trace requested) and with
    every layer classified in full (trace requested)."""
    from paper_2011_05749_b200 import DsfftConfig, SampleLedger, _device
    from paper_2011_05749_b200.dsfft import _dsfft_arrays

    if probe0 is not None:
        monkeypatch.setenv("AFFT_DSFFT_PROBE0", str(probe0))
    xd = _device.as_device_signal(dsfft_signal(case))
    cfg = DsfftConfig(mode=case["mode"], seed=case["seed"], noise_std=case["noise_std"])
    small = case["n"] <= 1 << 20  # the host ledger replay of a 2^24 decode is slow
    led_lazy = SampleLedger(case["n"]) if small else None
    led_full = SampleLedger(case["n"]) if small else None
    lazy = _dsfft_arrays(xd, case["k"], cfg, led_lazy)
    full = _dsfft_arrays(xd, case["k"], cfg, led_full, trace=[])
    if small:  # the ledger models the reference's reads: one classify per layer either way
        assert (led_lazy.count, led_lazy.unique_count) == (led_full.count, led_full.unique_count)
    return lazy, full


@pytest.mark.parametrize("probe0", [None, 1, 4096])
def test_probe_classifies_change_nothing(golden_dsfft, monkeypatch, probe0):
    """Intermediate layers' entries are discarded by the reference, so a noisy decode
    classifies only probe sets there (the active children of the multi-tons found one
    layer up; the first layer's first AFFT_DSFFT_PROBE0 buckets) and the whole layer only
    when a probe finds no multi-ton.  The entries — positions in insertion order and
    values — must be bit-identical to classifying every layer in full, for every golden
    case and config 4's signals, whatever the first probe's size (1: the chain dies out
    early and the full fallback runs often; 4096: the first layer in full)."""
    cases = [c for c in golden_dsfft["cases"] if c["mode"] != "exact"]
    cases += [json.load(open(p)) for p in C4]
    assert cases
    for case in cases:
        (pl, vl), (pf, vf) = _entries_lazy_and_full(case, monkeypatch, probe0)
        assert pl.tolist() == pf.tolist()
        assert np.array_equal(vl, vf)


def test_fused_spectrum_layers_change_nothing(golden_dsfft, monkeypatch):
    """The spectrum's last radix-256 pass decides the deepest nine full layers in its
    epilogue (bucketize.cu deep_fuse_epilogue, n = 2^24 at config 4) instead of a
    separate pass over Y; the sums run in the same order, so the layer traces and the
    entries must be bit-identical to the unfused path (AFFT_DSFFT_FUSE=0)."""
    from paper_2011_05749_b200 import DsfftConfig, _device
    from paper_2011_05749_b200.dsfft import _dsfft_arrays

    cases = [c for c in golden_dsfft["cases"] if c["mode"] != "exact"]
    cases += [json.load(open(p)) for p in C4]
    for case in cases:
        xd = _device.as_device_signal(dsfft_signal(case))
        cfg = DsfftConfig(mode=case["mode"], seed=case["seed"], noise_std=case["noise_std"])
        got = {}
        for fuse in ("1", "0"):
            monkeypatch.setenv("AFFT_DSFFT_FUSE", fuse)
            tr = []
            got[fuse] = (_dsfft_arrays(xd, case["k"], cfg, trace=tr), tr)
        (p1, v1), t1 = got["1"]
        (p0, v0), t0 = got["0"]
        assert t1 == t0
        assert p1.tolist() == p0.tolist()
        assert np.array_equal(v1, v0)


@pytest.mark.parametrize("n,k", [(1 << 16, 64), (1 << 16, 512), (1 << 24, 1024),
                                 (1 << 24, 256)])
def test_fused_layers_other_shapes(monkeypatch, n, k):
    """The fused epilogue at the other plan shapes it serves: n = 2^16 (two radix-256
    passes) with the stop layer below the fused depths (tree levels from the depth-8
    values) and above them (k = 512: depth 9, no shallower layer), and n = 2^24 with a
    stop layer at depth 10.  Layer traces and entries bit-identical to the unfused path."""
    from paper_2011_05749_b200 import DsfftConfig, _device, generate_test_case
    from paper_2011_05749_b200.dsfft import _dsfft_arrays

    snr = 20.0
    x = generate_test_case(n, k, snr, seed=77).signal.astype(np.complex64)
    xd = _device.as_device_signal(x)
    cfg = DsfftConfig(mode="noisy", seed=3, noise_std=float(np.sqrt(k * 10 ** (-snr / 10))))
    got = {}
    for fuse in ("1", "0"):
        monkeypatch.setenv("AFFT_DSFFT_FUSE", fuse)
        tr = []
        got[fuse] = (_dsfft_arrays(xd, k, cfg, trace=tr), tr)
    (p1, v1), t1 = got["1"]
    (p0, v0), t0 = got["0"]
    assert t1 == t0
    assert p1.tolist() == p0.tolist()
    assert np.array_equal(v1, v0)
    assert len(p1) > k // 2
