import os, sys, time, ctypes
import numpy as np, torch
ROOT = os.getcwd(); sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tools"))
from bench_suite import make_batch
from paper_2011_05749_b200 import DsfftConfig, _lib
import paper_2011_05749_b200.dsfft
D = sys.modules["paper_2011_05749_b200.dsfft"]
n, k, snr = 1 << 24, 4096, 20.0
x, _ = make_batch(n, k, snr, 2, torch.complex64, torch.device("cuda", 0), chunk=2)
cfg = DsfftConfig(mode="noisy", seed=0, noise_std=float(np.sqrt(k * 10 ** (-snr / 10))))
D.dsfft_device(x[0], k, cfg); torch.cuda.synchronize()
orig = _lib.load().afft_dsfft
acc = {"native": 0.0}
class Wrap:
    def __getattr__(self, name):
        return getattr(_lib.load.__wrapped__() if hasattr(_lib.load, "__wrapped__") else LIB, name)
LIB = _lib.load()
def timed(*a):
    t = time.perf_counter(); r = orig(*a); acc["native"] += time.perf_counter() - t; return r
class L:
    def __getattr__(self, nm):
        return timed if nm == "afft_dsfft" else getattr(LIB, nm)
_lib_load = _lib.load
_lib.load = lambda: L()
for rep in range(3):
    acc["native"] = 0.0
    t0 = time.perf_counter(); D._search_plan(n, cfg.seed); D._dt3_shift_table(n, cfg); t1 = time.perf_counter()
    tr0 = time.perf_counter(); D.dsfft_device(x[1], k, cfg); torch.cuda.synchronize(); tot = time.perf_counter() - tr0
    print(f"total {tot*1e3:.2f} ms; native {acc['native']*1e3:.2f}; numpy inputs {(t1-t0)*1e3:.2f}; rest {(tot-acc['native']-(t1-t0))*1e3:.2f}", flush=True)
