"""afft_dsfft_batch (C ABI, lockstep) at config 4: signals per call x worker streams.
python tools/dsfft_lockstep_sweep.py [snr]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from bench_suite import make_batch  # noqa: E402
from paper_2011_05749_b200 import DsfftConfig  # noqa: E402
from paper_2011_05749_b200.dsfft import _dsfft_batch_native, _on_worker_streams  # noqa: E402

snr = float(sys.argv[1]) if len(sys.argv) > 1 else 20.0
S, n, k = 32, 1 << 24, 4096
x, _ = make_batch(n, k, snr, S, torch.complex64, torch.device("cuda", 0), chunk=4)
cfgs = [DsfftConfig(mode="noisy", seed=i, noise_std=float(np.sqrt(k * 10 ** (-snr / 10))))
        for i in range(S)]


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


for streams, chunk in ((1, 32), (2, 16), (2, 8), (4, 8), (4, 4), (8, 4), (3, 11), (6, 6), (8, 2)):
    parts = [list(range(c0, min(S, c0 + chunk))) for c0 in range(0, S, chunk)]
    ms = timed(lambda: _on_worker_streams(
        x, parts, streams, lambda part: _dsfft_batch_native(x, k, cfgs, part)))
    print(f"snr {snr:g} streams {streams} x chunk {chunk}: {ms:.2f} ms per {S} = "
          f"{S / ms * 1e3:.0f} signals/s", flush=True)
