"""DSFFT in lockstep over a batch (afft_dsfft_batch): the same decisions as the
per-signal native loop — config-4 goldens from the reference decoded as one mixed-SNR
batch, and a synthetic batch compared signal by signal with the per-signal path."""

import glob
import json
import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN_DIR, cx, dsfft_signal

pytestmark = pytest.mark.gpu


def _configs(cases):
    from paper_2011_05749_b200 import DsfftConfig

    return [DsfftConfig(mode=c["mode"], seed=c["seed"], noise_std=c["noise_std"]) for c in cases]


def test_config4_goldens_in_one_lockstep_batch():
    from paper_2011_05749_b200.dsfft import _dsfft_batch_native, _top_k

    paths = sorted(glob.glob(os.path.join(GOLDEN_DIR, "golden_dsfft_c4_*db*.json")))
    cases = [json.load(open(p)) for p in paths]
    xs = torch.stack([torch.from_numpy(dsfft_signal(c)) for c in cases]).cuda()
    k, n = cases[0]["k"], cases[0]["n"]
    got = _dsfft_batch_native(xs, k, _configs(cases), list(range(len(cases))))
    assert sorted(got) == list(range(len(cases))), "a config-4 signal fell back"
    for i, c in enumerate(cases):
        out = _top_k(n, k, *got[i]).entries
        want = {f: cx(v) for f, v in c["truncated"]}
        assert set(out) == set(want), (paths[i], sorted(set(out) ^ set(want))[:10])
        assert max(abs(out[f] - v) for f, v in want.items()) <= 1e-6


def test_lockstep_equals_per_signal_path():
    from paper_2011_05749_b200 import DsfftConfig, dsfft_batch, generate_test_case

    n, k = 1 << 20, 256
    xs, cfgs = [], []
    for i, snr in enumerate((10.0, 20.0, 30.0, 20.0, 15.0, 25.0)):
        seed = 1000 + i
        xs.append(generate_test_case(n, k, snr, seed).signal.astype(np.complex64))
        cfgs.append(DsfftConfig(mode="noisy", seed=seed,
                                noise_std=float(np.sqrt(k * 10 ** (-snr / 10)))))
    xd = torch.from_numpy(np.stack(xs)).cuda()
    a = dsfft_batch(xd, k, cfgs, lockstep=True, chunk=4)
    b = dsfft_batch(xd, k, cfgs, lockstep=False)
    for i in range(len(xs)):
        assert list(a[i].entries) == list(b[i].entries), i
        assert max(abs(a[i].entries[f] - v) for f, v in b[i].entries.items()) == 0.0


def test_lockstep_equals_per_signal_path_c128_mixed():
    """complex128 input, mixed noise levels and seeds, plus an exact-mode signal (which
    leaves the lockstep path and is decoded alone): lockstep and per-signal decodes agree
    entry for entry."""
    from paper_2011_05749_b200 import DsfftConfig, dsfft_batch, generate_test_case

    n, k = 1 << 20, 256
    xs, cfgs = [], []
    for i, snr in enumerate((10.0, 30.0, "exact", 20.0)):
        seed = 2000 + i
        xs.append(generate_test_case(n, k, snr, seed).signal)
        if snr == "exact":
            cfgs.append(DsfftConfig(mode="exact", seed=seed))
        else:
            cfgs.append(DsfftConfig(mode="noisy", seed=seed,
                                    noise_std=float(np.sqrt(k * 10 ** (-snr / 10)))))
    xd = torch.from_numpy(np.stack(xs)).cuda()
    a = dsfft_batch(xd, k, cfgs, lockstep=True, chunk=3)
    b = dsfft_batch(xd, k, cfgs, lockstep=False)
    for i in range(len(xs)):
        assert list(a[i].entries) == list(b[i].entries), i
        assert max(abs(a[i].entries[f] - v) for f, v in b[i].entries.items()) == 0.0
