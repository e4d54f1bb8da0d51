"""Config-4 DSFFT throughput of dsfft_batch: per-signal worker streams against lockstep
chunks (afft_dsfft_batch) with several (streams, chunk) settings; every setting's spectra
are compared with the per-signal path's.

    python tools/dsfft_lockstep.py [signals] [streams:chunk,streams:chunk,...] [snr]
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from bench_suite import make_batch  # noqa: E402
from paper_2011_05749_b200 import DsfftConfig, dsfft_batch  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 32
sets = [tuple(int(v) for v in p.split(":")) for p in
        (sys.argv[2] if len(sys.argv) > 2 else "8:0,1:32,2:16,4:8").split(",")]
snr = float(sys.argv[3]) if len(sys.argv) > 3 else 20.0
n, k = 1 << 24, 4096
x, _ = make_batch(n, k, snr, S, torch.complex64, torch.device("cuda", 0), chunk=4)
cfg = DsfftConfig(mode="noisy", seed=0, noise_std=float(np.sqrt(k * 10 ** (-snr / 10))))
ref = dsfft_batch(x, k, cfg, streams=8)
torch.cuda.synchronize()
for streams, chunk in sets:
    kw = dict(streams=streams, lockstep=chunk > 0, chunk=max(1, chunk))
    dsfft_batch(x, k, cfg, **kw)
    torch.cuda.synchronize()
    best = None
    for _ in range(3):
        t = time.perf_counter()
        out = dsfft_batch(x, k, cfg, **kw)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t) * 1e3
        best = ms if best is None else min(best, ms)
    same = all(list(a.entries.items()) == list(b.entries.items()) for a, b in zip(out, ref))
    print(f"streams {streams} chunk {chunk}: {best:.1f} ms for {S} signals = "
          f"{S / best * 1e3:.1f} signals/s; identical to per-signal {same}", flush=True)
