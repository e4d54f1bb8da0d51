"""A small noisy DSFFT decode whose spectrum takes the fused last pass (n = 2^16, two
radix-256 passes), per-signal and in lockstep — for compute-sanitizer runs.
    compute-sanitizer --tool memcheck python tools/sanitize_dsfft.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_05749_b200 import DsfftConfig, _device, dsfft_batch, generate_test_case  # noqa
from paper_2011_05749_b200.dsfft import _dsfft_arrays  # noqa: E402

n, k, snr = 1 << 16, 64, 20.0
xs = [generate_test_case(n, k, snr, seed=s).signal.astype(np.complex64) for s in range(4)]
cfg = DsfftConfig(mode="noisy", seed=3, noise_std=float(np.sqrt(k * 10 ** (-snr / 10))))
p, v = _dsfft_arrays(_device.as_device_signal(xs[0]), k, cfg)
xd = torch.from_numpy(np.stack(xs)).cuda()
a = dsfft_batch(xd, k, cfg, streams=1, lockstep=True, chunk=4)
b = dsfft_batch(xd, k, cfg, streams=2)
torch.cuda.synchronize()
print("ok", len(p), all(list(x.entries) == list(y.entries) for x, y in zip(a, b)))
