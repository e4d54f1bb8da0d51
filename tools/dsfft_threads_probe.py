"""Where dsfft_batch's worker threads spend their time (diagnostic): per signal, the
Python work before the native call, the native layer loop (afft_dsfft, GIL released),
and the Python work after it, plus the wall time of the whole batch.

    python tools/dsfft_threads_probe.py [streams] [signals]
"""
import os
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from bench_suite import make_batch  # noqa: E402
from paper_2011_05749_b200 import DsfftConfig, _lib, dsfft_batch  # noqa: E402
import paper_2011_05749_b200.dsfft  # noqa: E402,F401

D = sys.modules["paper_2011_05749_b200.dsfft"]
streams = int(sys.argv[1]) if len(sys.argv) > 1 else 4
S = int(sys.argv[2]) if len(sys.argv) > 2 else 16
n, k, snr = 1 << 24, 4096, 20.0
x, _ = make_batch(n, k, snr, S, torch.complex64, torch.device("cuda", 0), chunk=4)
cfg = DsfftConfig(mode="noisy", seed=0, noise_std=float(np.sqrt(k * 10 ** (-snr / 10))))

lib = _lib.load()
native = lib.afft_dsfft
rec = {}
lock = threading.Lock()


def timed_native(*a):
    t0 = time.perf_counter()
    rc = native(*a)
    t1 = time.perf_counter()
    with lock:
        rec.setdefault(threading.get_ident(), []).append(("native", t0, t1))
    return rc


orig = D.dsfft


def timed_dsfft(*a, **kw):
    t0 = time.perf_counter()
    out = orig(*a, **kw)
    t1 = time.perf_counter()
    with lock:
        rec.setdefault(threading.get_ident(), []).append(("call", t0, t1))
    return out


lib.afft_dsfft = timed_native
D.dsfft = timed_dsfft
dsfft_batch(x, k, cfg, streams=streams)  # warm (pool threads, streams, memory pool)
torch.cuda.synchronize()
rec.clear()
t = time.perf_counter()
dsfft_batch(x, k, cfg, streams=streams)
torch.cuda.synchronize()
wall = time.perf_counter() - t
calls = [e for v in rec.values() for e in v if e[0] == "call"]
nats = [e for v in rec.values() for e in v if e[0] == "native"]
call_ms = sum(e[2] - e[1] for e in calls) * 1e3 / len(calls)
nat_ms = sum(e[2] - e[1] for e in nats) * 1e3 / len(nats)
print(f"streams {streams}, {S} signals: {wall * 1e3:.1f} ms = {S / wall:.1f} signals/s; per signal "
      f"call {call_ms:.2f} ms, native {nat_ms:.2f} ms, python {call_ms - nat_ms:.2f} ms; "
      f"threads {len(rec)}")
