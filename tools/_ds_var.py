import os, sys, time
import numpy as np, torch
ROOT = os.getcwd(); sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tools"))
from bench_suite import make_batch
from paper_2011_05749_b200 import DsfftConfig, dsfft_batch
n, k, snr, S = 1 << 24, 4096, 20.0, 16
x, _ = make_batch(n, k, snr, S, torch.complex64, torch.device("cuda", 0), chunk=4)
cfg = DsfftConfig(mode="noisy", seed=0, noise_std=float(np.sqrt(k * 10 ** (-snr / 10))))
for streams in (4, 8, 4, 8, 4, 8, 16, 16):
    torch.cuda.synchronize(); t = time.perf_counter()
    dsfft_batch(x, k, cfg, streams=streams); torch.cuda.synchronize()
    ms = (time.perf_counter() - t) * 1e3
    print(f"streams {streams}: {ms:.1f} ms for {S} = {S / ms * 1e3:.1f}/s", flush=True)
