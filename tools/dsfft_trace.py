"""Layer trace of config-4 DSFFT decodes (diagnostic): which depths are expanded and
classified, with how many active buckets / multitons, per SNR."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from bench_suite import make_batch  # noqa: E402
from paper_2011_05749_b200 import DsfftConfig  # noqa: E402
import paper_2011_05749_b200.dsfft  # noqa: E402,F401

D = sys.modules["paper_2011_05749_b200.dsfft"]
n, k = 1 << 24, 4096
for snr in (10.0, 20.0, 30.0):
    x, _ = make_batch(n, k, snr, 2, torch.complex64, torch.device("cuda", 0), chunk=2)
    cfg = DsfftConfig(mode="noisy", seed=0, noise_std=float(np.sqrt(k * 10 ** (-snr / 10))))
    for s in range(2):
        tr = []
        D.dsfft_device(x[s], k, cfg, trace=tr)
        print(f"snr {snr:.0f} signal {s}: {tr}")
