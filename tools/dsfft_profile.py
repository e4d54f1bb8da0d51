"""Per-stage wall time of one config-4 DSFFT decode (diagnostic; synchronises per stage)."""

import collections
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

acc = collections.defaultdict(float)
cnt = collections.Counter()


def wrap(name):
    fn = getattr(D, name)

    def inner(*a, **k):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = fn(*a, **k)
        torch.cuda.synchronize()
        acc[name] += time.perf_counter() - t
        cnt[name] += 1
        return r

    setattr(D, name, inner)


for name in ("_initial", "_expand", "_classify", "_resolve_aliased", "_rows", "_active",
             "_full_values"):
    wrap(name)

n, k, snr = 1 << 24, 4096, 20.0
x, _ = make_batch(n, k, snr, 2, torch.complex64, torch.device("cuda", 0), chunk=2)
cfg = DsfftConfig(mode="noisy", seed=0, noise_std=float(np.sqrt(k * 10 ** (-snr / 10))))
D.dsfft_device(x[0], k, cfg)
acc.clear()
cnt.clear()
torch.cuda.synchronize()
t0 = time.perf_counter()
D.dsfft_device(x[1], k, cfg)
torch.cuda.synchronize()
total = time.perf_counter() - t0
print(f"total {total * 1e3:.1f} ms")
for name, v in sorted(acc.items(), key=lambda kv: -kv[1]):
    print(f"  {name:18s} {v * 1e3:8.2f} ms  x{cnt[name]}")

# ---- per C-ABI entry point (synchronised wall time per call)
from paper_2011_05749_b200 import _lib  # noqa: E402

lib = _lib.load()
cacc = collections.defaultdict(float)
ccnt = collections.Counter()


class Timed:
    def __init__(self, fn, name):
        self.fn, self.name = fn, name

    def __call__(self, *a):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = self.fn(*a)
        torch.cuda.synchronize()
        cacc[self.name] += time.perf_counter() - t
        ccnt[self.name] += 1
        return r


for name in list(_lib.SIGNATURES):
    setattr(lib, name, Timed(getattr(lib, name), name))
torch.cuda.synchronize()
t0 = time.perf_counter()
D.dsfft_device(x[1], k, cfg)
torch.cuda.synchronize()
print(f"total (C calls synchronised) {(time.perf_counter() - t0) * 1e3:.1f} ms")
for name, v in sorted(cacc.items(), key=lambda kv: -kv[1]):
    print(f"  {name:32s} {v * 1e3:8.2f} ms  x{ccnt[name]}")
