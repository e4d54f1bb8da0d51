"""One warm lockstep DSFFT batch (afft_dsfft_batch) of config-4 signals between
cudaProfilerStart/Stop (for ncu launch lists).  python tools/dsfft_lockstep_one.py [S]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from bench_suite import make_batch  # noqa: E402
from paper_2011_05749_b200 import DsfftConfig  # noqa: E402
from paper_2011_05749_b200.dsfft import _dsfft_batch_native  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 8
n, k, snr = 1 << 24, 4096, 20.0
x, _ = make_batch(n, k, snr, S, torch.complex64, torch.device("cuda", 0), chunk=4)
cfgs = [DsfftConfig(mode="noisy", seed=i, noise_std=float(np.sqrt(k * 10 ** (-snr / 10))))
        for i in range(S)]
_dsfft_batch_native(x, k, cfgs, list(range(S)))
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
import time
t = time.perf_counter()
out = _dsfft_batch_native(x, k, cfgs, list(range(S)))
torch.cuda.synchronize()
print("wall ms", (time.perf_counter() - t) * 1e3, "decoded", len(out))
torch.cuda.cudart().cudaProfilerStop()
