"""Config-4 DSFFT throughput vs concurrent streams (dsfft_batch(streams=S)): with the
layer loop native, ctypes releases the GIL for the whole decode, so several signals'
loops overlap their read-back latencies.  Checks that every stream count returns the
same spectra as the sequential run.

    python tools/dsfft_streams.py [signals] [streams,streams,...]"""
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

n, k, snr = 1 << 24, 4096, 20.0
S = int(sys.argv[1]) if len(sys.argv) > 1 else 8
STREAMS = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 2, 4, 8, 1]
x, _ = make_batch(n, k, snr, S, torch.complex64, torch.device("cuda", 0), chunk=4)
cfg = DsfftConfig(mode="noisy", seed=0, noise_std=float(np.sqrt(k * 10 ** (-snr / 10))))
ref = None
for streams in STREAMS:
    dsfft_batch(x, k, cfg, streams=streams)
    torch.cuda.synchronize()
    t = time.perf_counter()
    out = dsfft_batch(x, k, cfg, streams=streams)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t) * 1e3
    same = ref is None or all(a.entries == b.entries for a, b in zip(out, ref))
    ref = ref or out
    print(f"streams {streams}: {ms:.1f} ms for {S} signals = {S / ms * 1e3:.1f} signals/s; "
          f"identical {same}", flush=True)
