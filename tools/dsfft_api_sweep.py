"""dsfft_batch (the drop-in API, SparseSpectrum dicts included) at config 4, 20 dB:
per-signal loops against lockstep chunks of several sizes / stream counts.
python tools/dsfft_api_sweep.py"""
import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tools"))
from bench_suite import make_batch
from paper_2011_05749_b200 import DsfftConfig, dsfft_batch
snr = 20.0
S, n, k = 32, 1 << 24, 4096
x, _ = make_batch(n, k, snr, S, torch.complex64, torch.device("cuda", 0), chunk=4)
cfgs = [DsfftConfig(mode="noisy", seed=i, noise_std=float(np.sqrt(k * 10 ** (-snr / 10)))) for i in range(S)]
def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps
for kw in (dict(lockstep=False), dict(), dict(chunk=3), dict(chunk=2), dict(chunk=4, streams=6),
           dict(chunk=4, streams=12), dict(chunk=2, guided=False), dict(chunk=8)):
    ms = timed(lambda: dsfft_batch(x, k, cfgs, **kw))
    print(kw, f"{ms:.2f} ms per {S} = {S/ms*1e3:.0f} signals/s", flush=True)
