"""Where a config-4 DSFFT decode spends its wall time (diagnostic): the host-side
numpy inputs (search plan, DT3 shift table), the native layer loop (afft_dsfft), and
the ledger/trace replay.  Compare with the GPU busy time from an ncu launch list of
tools/dsfft_one.py."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from bench_suite import make_batch  # noqa: E402
from paper_2011_05749_b200 import DsfftConfig  # noqa: E402
import paper_2011_05749_b200.dsfft  # noqa: E402,F401

D = sys.modules["paper_2011_05749_b200.dsfft"]
n, k, snr = 1 << 24, 4096, 20.0
x, _ = make_batch(n, k, snr, 2, torch.complex64, torch.device("cuda", 0), chunk=2)
cfg = DsfftConfig(mode="noisy", seed=0, noise_std=float(np.sqrt(k * 10 ** (-snr / 10))))
D.dsfft_device(x[0], k, cfg)
torch.cuda.synchronize()
reps = 5
t = time.perf_counter()
for _ in range(reps):
    D._search_plan(n, cfg.seed)
    D._dt3_shift_table(n, cfg)
prep = (time.perf_counter() - t) / reps
t = time.perf_counter()
for _ in range(reps):
    D.dsfft_device(x[1], k, cfg)
torch.cuda.synchronize()
total = (time.perf_counter() - t) / reps
print(f"dsfft_device {total * 1e3:.2f} ms/signal; numpy inputs {prep * 1e3:.2f} ms; "
      f"native loop + replay {(total - prep) * 1e3:.2f} ms")
