"""Edge cases of the device paths: strided and misaligned rows, empty batches, k = 0,
graphs too large for shared memory (global-scratch fallback), bucket counts on the
four-step DFT path — each checked against the oracle."""

import numpy as np
import pytest
import torch

from oracle import ffast as of

pytestmark = pytest.mark.gpu


def _signals(n, k, count, seed0=0, dtype=np.complex128):
    from paper_2011_05749_b200 import generate_test_case

    return np.stack([generate_test_case(n, k, "exact", seed0 + i).signal for i in range(count)]
                    ).astype(dtype)


def test_strided_rows_equal_contiguous():
    from paper_2011_05749_b200 import ffast_batch

    n, k, f = 4095, 8, [63, 65]
    xs = _signals(n, k, 5)
    wide = torch.zeros((5, n + 37), dtype=torch.complex128, device="cuda")
    wide[:, :n] = torch.from_numpy(xs).cuda()
    strided = wide[:, :n]  # ld = n + 37
    assert strided.stride(0) == n + 37
    a = ffast_batch(strided, k, f)
    b = ffast_batch(torch.from_numpy(xs).cuda(), k, f)
    for i in range(5):
        assert a.full_spectrum(i).entries == b.full_spectrum(i).entries


def test_misaligned_complex64_rows():
    """n odd => every other c64 row starts 8 bytes off a 16-byte boundary (stream head path)."""
    from paper_2011_05749_b200 import ffast_batch

    n, k, f = 4095, 8, [63, 65]
    xs = _signals(n, k, 6, seed0=10, dtype=np.complex64)
    for mode in ("0", "1", "2", "3", "4"):
        import os

        os.environ["AFFT_FFAST_MODE"] = mode
        try:
            res = ffast_batch(torch.from_numpy(xs).cuda(), k, f)
        finally:
            del os.environ["AFFT_FFAST_MODE"]
        for i in range(6):
            _, o = of.ffast(xs[i].astype(np.complex128), k, f)
            assert list(res.full_spectrum(i).entries) == list(o["recovered"])


@pytest.mark.parametrize("parts", ["", "12", "16"])
def test_split_streams_small_norm_parts(parts):
    """Mode 4 with fewer norm-pass parts than CTAs per signal (c128 n = 32,760 gives
    nparts = 8 while mode 4 runs up to 12, or 16 by override): its partial sums and
    tickets must stay inside the workspace afft_ffast_workspace_size reports.  The
    workspace is followed by a guard band that must come back untouched."""
    import os

    from paper_2011_05749_b200 import _lib, ffast_batch
    from paper_2011_05749_b200.batch import ffast_workspace_bytes

    n, k, f, batch = 32760, 8, [13, 35, 72], 64
    lib = _lib.load()
    assert 2 <= int(lib.afft_sumsq_parts(n, _lib.AFFT_C128)) <= 12
    xs = _signals(n, k, batch, seed0=40)
    need = ffast_workspace_bytes(n, _lib.AFFT_C128, batch, f)
    buf = torch.full((need + 4096,), 0xA5, dtype=torch.uint8, device="cuda")
    os.environ["AFFT_FFAST_MODE"] = "4"
    if parts:
        os.environ["AFFT_FFAST_PARTS"] = parts
    try:
        res = ffast_batch(torch.from_numpy(xs).cuda(), k, f, workspace=buf[:need])
        torch.cuda.synchronize()
    finally:
        os.environ.pop("AFFT_FFAST_MODE", None)
        os.environ.pop("AFFT_FFAST_PARTS", None)
    assert bool((buf[need:] == 0xA5).all()), "mode 4 wrote past its workspace"
    for i in range(batch):
        _, o = of.ffast(xs[i], k, f)
        assert list(res.full_spectrum(i).entries) == list(o["recovered"])


def test_empty_and_k0():
    from paper_2011_05749_b200 import ffast, ffast_batch

    res = ffast_batch(torch.zeros((0, 4095), dtype=torch.complex128, device="cuda"), 4, [63, 65])
    assert res.count.numel() == 0
    x = _signals(4095, 4, 1)[0]
    assert ffast(x, 0).entries == {}
    res = ffast_batch(x[None, :], 0, [63, 65])
    assert int(res.count[0]) == 0 and int(res.all_count[0]) > 0  # decoded, then truncated to 0


def test_large_graph_fallback_and_four_step():
    """b = 8192 > 4096: four-step graph build, global-memory peeling scratch, large truncation."""
    from paper_2011_05749_b200 import CyclePlan, ffast, plan_cycles

    n, k = 8192 * 5, 6
    plan, _ = plan_cycles(n, k, "exact")
    assert max(plan.factors) > 4096
    for seed in range(3):
        x = _signals(n, k, 1, seed0=seed)[0]
        out = ffast(x, k, plan=CyclePlan(plan.factors, [0, 1, 2]))
        trunc, o = of.ffast(x, k, plan.factors)
        assert set(out.entries) == set(trunc)
        for f, v in trunc.items():
            assert abs(out.entries[f] - v) < 1e-9


def test_peel_decode_resumes_with_prior_recovered():
    """peel_decode on a graph that already holds recovered tones (peeling.py:281-282 default
    max_rounds = len(recovered) + 8; prior entries must not be re-harvested)."""
    from paper_2011_05749_b200 import CyclePlan, generate_test_case, peel_decode
    from paper_2011_05749_b200.peeling import build_graph, exact_thresholds

    case = generate_test_case(504, 6, "exact", seed=2)
    g = build_graph(case.signal, CyclePlan([7, 8, 9], [0, 1, 2]))
    e = exact_thresholds(case.signal)
    r1 = peel_decode(g, "exact", eps_zero=e, eps_ratio=e, max_rounds=1)
    first = dict(g.recovered)
    r2 = peel_decode(g, "exact", eps_zero=e, eps_ratio=e)
    assert list(g.recovered)[: len(first)] == list(first)
    g_all = build_graph(case.signal, CyclePlan([7, 8, 9], [0, 1, 2]))
    r_all = peel_decode(g_all, "exact", eps_zero=e, eps_ratio=e, max_rounds=12)
    assert set(r2.spectrum.entries) == set(r_all.spectrum.entries)
    assert r1.rounds == 1
