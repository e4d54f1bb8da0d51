"""Reentrancy per CUDA stream: the same calls issued concurrently from several host
threads, each on its own stream, give exactly the sequential results.  (Regression:
kernels' dynamic shared-memory limits are process-wide attributes; a thread setting a
smaller limit could invalidate another thread's launch.)"""

import threading

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _jobs():
    from paper_2011_05749_b200 import (DsfftConfig, OneShotConfig, dsfft, ffast,
                                       generate_test_case, r_ffast, sfft_dt)
    from paper_2011_05749_b200.bucketize import bucketize_device

    cases = {
        "ffast": generate_test_case(4095, 8, "exact", seed=1).signal,
        "rffast": generate_test_case(4095, 4, 15.0, seed=2).signal,
        "dt3": generate_test_case(1 << 14, 8, "exact", seed=3).signal,
        "dsfft": generate_test_case(1 << 16, 8, 20.0, seed=4).signal,
        "big": np.random.default_rng(5).normal(size=1 << 18) + 0j,
    }
    return [
        lambda: sorted(ffast(cases["ffast"], 8).entries.items()),
        lambda: sorted(r_ffast(cases["rffast"], 4, seed=2, snr_hint=15.0).entries.items()),
        lambda: sorted(sfft_dt(cases["dt3"], 8, OneShotConfig.default(1 << 14, 8, "dt3", 3))
                       .entries.items()),
        lambda: sorted(dsfft(cases["dsfft"], 8, DsfftConfig(mode="noisy", seed=4,
                                                            noise_std=0.08)).entries.items()),
        # large-b DFTs of different sizes (different dynamic smem per launch)
        lambda: bucketize_device(torch.from_numpy(cases["big"]).cuda(), 1 << 16, [0, 5])
        .cpu().numpy().tolist(),
        lambda: bucketize_device(torch.from_numpy(cases["big"]).cuda(), 3 << 13, [1])
        .cpu().numpy().tolist() if (1 << 18) % (3 << 13) == 0 else None,
        lambda: bucketize_device(torch.from_numpy(cases["big"]).cuda(), 1 << 13, [7])
        .cpu().numpy().tolist(),
    ]


def test_concurrent_streams_match_sequential():
    jobs = _jobs()
    want = [job() for job in jobs]
    for _ in range(3):
        got = [None] * len(jobs)
        errors = []

        def run(i):
            try:
                s = torch.cuda.Stream()
                with torch.cuda.stream(s):
                    got[i] = jobs[i]()
                s.synchronize()
            except Exception as exc:  # noqa: BLE001 - reported below
                errors.append(exc)

        threads = [threading.Thread(target=run, args=(i,)) for i in range(len(jobs))]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        assert not errors, errors
        assert got == want
