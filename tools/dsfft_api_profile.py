"""Where dsfft_batch's wall time goes at config 4 (diagnostic): per-call native time
(afft_dsfft_batch / afft_dsfft, AFFT_DSFFT_PROFILE), the Python-side truncation and dict
building, for the per-signal and lockstep forms.
    python tools/dsfft_api_profile.py [signals]"""
import cProfile
import os
import pstats
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from bench_suite import make_batch  # noqa: E402
from paper_2011_05749_b200 import DsfftConfig, dsfft_batch  # noqa: E402
from paper_2011_05749_b200.dsfft import _top_k  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 32
n, k, snr = 1 << 24, 4096, 20.0
x, _ = make_batch(n, k, snr, S, torch.complex64, torch.device("cuda", 0), chunk=4)
cfg = DsfftConfig(mode="noisy", seed=0, noise_std=float(np.sqrt(k * 10 ** (-snr / 10))))
out = dsfft_batch(x, k, cfg)
pos = np.array(list(out[0].entries), dtype=np.int64)
val = np.array(list(out[0].entries.values()), dtype=np.complex128)
pos = np.concatenate([pos, pos + n // 2])[: 5000] % n
val = np.concatenate([val, val * 0.5])[: 5000]
t = time.perf_counter()
for _ in range(100):
    _top_k(n, k, pos, val)
print(f"_top_k of 5000 entries: {(time.perf_counter() - t) * 10:.3f} ms")
for kw in (dict(streams=8), dict(streams=4, lockstep=True, chunk=8),
           dict(streams=2, lockstep=True, chunk=16)):
    dsfft_batch(x, k, cfg, **kw)
    torch.cuda.synchronize()
    t = time.perf_counter()
    dsfft_batch(x, k, cfg, **kw)
    torch.cuda.synchronize()
    print(kw, f"{(time.perf_counter() - t) * 1e3:.1f} ms for {S}")
    pr = cProfile.Profile()
    pr.enable()
    dsfft_batch(x, k, cfg, **kw)
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(8)
