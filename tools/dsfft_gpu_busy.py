"""GPU busy fraction of dsfft_batch (diagnostic): the union of all kernel intervals
(torch.profiler / CUPTI sees the library's kernels too) against the wall time of the
batch, and the summed kernel time per signal.

    python tools/dsfft_gpu_busy.py [streams] [signals] [lockstep 0/1] [chunk]
"""
import os
import sys
import time

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from bench_suite import make_batch  # noqa: E402
from paper_2011_05749_b200 import DsfftConfig, dsfft_batch  # noqa: E402

streams = int(sys.argv[1]) if len(sys.argv) > 1 else 4
S = int(sys.argv[2]) if len(sys.argv) > 2 else 16
lock = (sys.argv[3] != "0") if len(sys.argv) > 3 else True
chunk = int(sys.argv[4]) if len(sys.argv) > 4 else 8
n, k, snr = 1 << 24, 4096, 20.0
x, _ = make_batch(n, k, snr, S, torch.complex64, torch.device("cuda", 0), chunk=4)
cfg = DsfftConfig(mode="noisy", seed=0, noise_std=float(np.sqrt(k * 10 ** (-snr / 10))))
dsfft_batch(x, k, cfg, streams=streams, lockstep=lock, chunk=chunk)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    t = time.perf_counter()
    dsfft_batch(x, k, cfg, streams=streams, lockstep=lock, chunk=chunk)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t
iv = []
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.elapsed_us() > 0:
        iv.append((e.time_range.start, e.time_range.end))
iv.sort()
busy, cur_s, cur_e, ksum = 0.0, None, None, 0.0
for s, e in iv:
    ksum += e - s
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
if cur_e is not None:
    busy += cur_e - cur_s
span = (iv[-1][1] - iv[0][0]) if iv else 0
print(f"lockstep {lock} chunk {chunk}, streams {streams}, {S} signals: wall {wall * 1e3:.1f} ms ({S / wall:.0f} signals/s), "
      f"kernel span {span / 1e3:.1f} ms, GPU busy {busy / 1e3:.1f} ms "
      f"({100 * busy / max(span, 1):.0f}% of the span), summed kernel time "
      f"{ksum / 1e3 / S:.2f} ms per signal, {len(iv)} kernels")
