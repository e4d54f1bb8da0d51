"""GPU bucketization (gather + small DFT) against the reference goldens and the oracle.

Mirrors the reference's tests/test_bucketize.py: exhaustive alias sums at small
n, single-tone residues, linearity, ledger accounting — plus config-shaped
stages (b = 49..51, 127..129, 1024 with the sFFT-DT structured shifts).
Tolerance: 1e-12 relative to the largest bucket magnitude (complex128
arithmetic; the DFT differs from pocketfft only in rounding).
"""

import numpy as np
import pytest
import torch

from conftest import cx, golden_signal
from oracle import ffast as of

pytestmark = pytest.mark.gpu


def _close(got, want, rel=1e-12):
    scale = max(1.0, float(np.max(np.abs(want))))
    return float(np.max(np.abs(np.asarray(got) - np.asarray(want)))) <= rel * scale


def test_goldens(golden_ffast):
    from paper_2011_05749_b200 import bucketize

    for case in golden_ffast["bucketize"]:
        if "x" in case:
            x = np.array([cx(v) for v in case["x"]])
        else:
            x = golden_signal(case["gen"])  # complex64 stays complex64 on the device
        got = bucketize(x, case["b"], case["tau"]).values
        want = np.array([cx(v) for v in case["values"]])
        assert _close(got, want), (case["b"], case["tau"])


def test_alias_sum_exhaustive_small(rng):
    from paper_2011_05749_b200 import bucketize_set, dense_dft

    for n in (8, 12, 20, 30, 49, 60):
        x = rng.normal(size=n) + 1j * rng.normal(size=n)
        dense = dense_dft(x)
        for b in [d for d in range(1, n + 1) if n % d == 0]:
            taus = list(range(-2, n + 2))
            got = bucketize_set(x, b, taus)
            for tau, sp in zip(taus, got):
                # alias sum: y[i] = sum_j X[j*b + i] * w^(tau*(j*b+i))
                f = np.arange(n)
                contrib = dense * np.exp(-2j * np.pi * ((tau * f) % n) / n)
                want = np.array([contrib[i::b].sum() for i in range(b)])
                assert np.allclose(sp.values, want, atol=1e-9)


@pytest.mark.parametrize("n,b", [(124950, 49), (124950, 50), (124950, 51), (2097024, 127),
                                 (2097024, 128), (2097024, 129), (1 << 22, 1024),
                                 (1 << 24, 4096), (511 * 512 * 8, 511), (3 * 17 * 19 * 73, 73 * 17),
                                 # K2' four-step path (b > 4096)
                                 (9728 * 7, 9728), (13797 * 5, 13797), (1 << 20, 1 << 13),
                                 (1 << 20, 1 << 20), (3 << 16, 3 << 15)])
def test_config_sizes_vs_oracle(n, b):
    from paper_2011_05749_b200.bucketize import bucketize_device

    rng = np.random.default_rng(n + b)
    x = (rng.normal(size=n) + 1j * rng.normal(size=n)).astype(np.complex128)
    shifts = [0, 1, 2, -4, 7, n - 1, 12345]
    got = bucketize_device(torch.from_numpy(x).cuda(), b, shifts).cpu().numpy()
    want = of.bucket_values(x, b, shifts)
    assert _close(got, want, 1e-12)


def test_complex64_input_upcasts_exactly():
    from paper_2011_05749_b200.bucketize import bucketize_device

    rng = np.random.default_rng(5)
    x = (rng.normal(size=129 * 64) + 1j * rng.normal(size=129 * 64)).astype(np.complex64)
    got = bucketize_device(torch.from_numpy(x).cuda(), 129, [0, 1, 2]).cpu().numpy()
    want = of.bucket_values(x.astype(np.complex128), 129, [0, 1, 2])
    assert _close(got, want, 1e-12)


def test_single_tone_residue_and_linearity(rng):
    from paper_2011_05749_b200 import SparseSpectrum, bucketize, inverse_dft

    n = 24
    for f in (0, 5, 17):
        x = inverse_dft(SparseSpectrum(n, {f: 1.0}))
        for b in (4, 6, 8):
            for tau in (0, 1, 7, -3):
                out = bucketize(x, b, tau).values
                assert abs(out[f % b] - np.exp(-2j * np.pi * ((tau * f) % n) / n)) < 1e-9
                assert np.max(np.abs(np.delete(out, f % b))) < 1e-9
    x = rng.normal(size=20) + 1j * rng.normal(size=20)
    y = rng.normal(size=20) + 1j * rng.normal(size=20)
    a, c = 2.0 - 1j, -0.5 + 3j
    comb = bucketize(a * x + c * y, 5, 3).values
    sep = a * bucketize(x, 5, 3).values + c * bucketize(y, 5, 3).values
    assert np.linalg.norm(comb - sep) <= 1e-9 * max(1.0, np.linalg.norm(sep))


def test_errors_and_ledger():
    from paper_2011_05749_b200 import SampleLedger, bucketize, bucketize_set

    with pytest.raises(ValueError):
        bucketize(np.zeros(10), 4, 0)
    ledger = SampleLedger(24)
    bucketize_set(np.zeros(24), 6, [0, 1, 2, 3, 10], ledger)
    assert ledger.count == 30 and ledger.unique_count <= 24


def test_large_b_batched_and_strided():
    """Four-step path with a batch, per-signal rows and the node layout."""
    from paper_2011_05749_b200 import _lib
    from paper_2011_05749_b200 import peeling

    rng = np.random.default_rng(7)
    n, factors, shifts = 9728 * 13 * 4, [9728, 13 * 4], [0, 1, 2, 5]
    xs = (rng.normal(size=(3, n)) + 1j * rng.normal(size=(3, n))).astype(np.complex64)
    for i in range(3):
        got = peeling.build_graph_device(torch.from_numpy(xs[i]).cuda(), factors, shifts)
        want = of.graph_values(xs[i].astype(np.complex128), factors, shifts)
        assert _close(got.cpu().numpy(), want, 1e-12)
    with pytest.raises(Exception):
        # prime bucket count above the one-CTA limit has no two-factor split
        from paper_2011_05749_b200.bucketize import bucketize_device
        bucketize_device(torch.zeros(4099 * 2, dtype=torch.complex128).cuda(), 4099, [0])


def test_device_input_synthesis_matches_host_model():
    """§8f item 1: device-synthesised inputs equal generate_test_case to ~1e-15."""
    from paper_2011_05749_b200.signals import generate_test_case, generate_test_case_device

    for n, k, snr, seed in [(124950, 40, "exact", 3), (1 << 16, 16, 20.0, 2), (4095, 4, 10.0, 0)]:
        ref = generate_test_case(n, k, snr, seed)
        x, truth = generate_test_case_device(n, k, snr, seed)
        assert truth.entries == ref.truth.entries
        d = np.max(np.abs(x.cpu().numpy() - ref.signal))
        assert d <= 1e-12 * max(1.0, np.max(np.abs(ref.signal))), d


@pytest.mark.parametrize("L", [1, 2, 8, 32])
def test_alias_rows_match_bucketize_rows(L):
    """afft_alias_rows (rows from the resident spectrum by the alias identity) equals
    afft_bucketize_rows (coset DFTs of the signal) for DSFFT's deep layers."""
    import torch

    from paper_2011_05749_b200 import _device, _lib

    n = 1 << 14
    b = n // L
    rng = np.random.default_rng(L)
    x = torch.from_numpy(rng.normal(size=n) + 1j * rng.normal(size=n)).cuda()
    shifts = [int(t) for t in rng.integers(-n, 2 * n, size=40)] + [0, 1, 2]
    idx = torch.from_numpy(np.sort(rng.choice(b, size=min(b, 300), replace=False))).cuda()
    lib = _lib.load()
    sp = _device.stream_ptr()
    sb, ns = _lib.host_i64(shifts)
    rows_ref = torch.empty((idx.numel(), len(shifts)), dtype=torch.complex128, device="cuda")
    en_ref = torch.empty(b, dtype=torch.float64, device="cuda")
    _lib.check(lib.afft_bucketize_rows(x.data_ptr(), 1, n, b, sb, ns, idx.data_ptr(), idx.numel(),
                                       rows_ref.data_ptr(), en_ref.data_ptr(), sp), "rows")
    Y = torch.empty(n, dtype=torch.complex128, device="cuda")
    s0, n0 = _lib.host_i64([0])
    _lib.check(lib.afft_bucketize(x.data_ptr(), 1, n, 1, n, n, s0, n0, Y.data_ptr(), n, n, 1, sp),
               "spectrum")
    rows = torch.empty_like(rows_ref)
    en = torch.empty_like(en_ref)
    v0 = torch.empty(b, dtype=torch.complex128, device="cuda")
    _lib.check(lib.afft_alias_rows(Y.data_ptr(), n, b, sb, ns, idx.data_ptr(), idx.numel(),
                                   rows.data_ptr(), en.data_ptr(), v0.data_ptr(), sp), "alias")
    scale = float(rows_ref.abs().max())
    assert float((rows - rows_ref).abs().max()) <= 1e-12 * scale
    assert torch.allclose(en, en_ref, rtol=1e-11, atol=0)
    ref0 = np.fft.fft(x.cpu().numpy()[::L]) / b
    assert np.allclose(v0.cpu().numpy(), ref0, rtol=0, atol=1e-12 * np.abs(ref0).max())


@pytest.mark.parametrize("b", [8186, 15015, 6480, 12288, 32766, 8168, 65536 * 3, 4097 * 2])
def test_large_b_mixed_radix_sizes(b):
    """K2' global passes at b > 4096 with mixed prime factors (radix groups <= 256, a
    prime above 256 as its own radix, 4097 = 17 * 241): against numpy on a shifted,
    subsampled signal."""
    import torch

    from paper_2011_05749_b200.bucketize import bucketize_device

    L = 3
    n = b * L
    rng = np.random.default_rng(b)
    x = rng.normal(size=n) + 1j * rng.normal(size=n)
    shifts = [0, 1, -7, n + 5]
    got = bucketize_device(torch.from_numpy(x).cuda(), b, shifts).cpu().numpy()
    for t, tau in enumerate(shifts):
        idx = (np.arange(b) * L - tau) % n
        want = np.fft.fft(x[idx]) / b
        assert np.max(np.abs(got[t] - want)) <= 1e-12 * np.max(np.abs(want)) * np.log2(b)
