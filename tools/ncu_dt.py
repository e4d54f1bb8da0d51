"""Small driver of config 2 (sFFT-DT2) / config 4 (DT3) for launch lists (diagnostic)."""

import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from bench_suite import case_seed, make_batch  # noqa: E402
from paper_2011_05749_b200 import sfft_dt_batch  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c2"
dev = torch.device("cuda", 0)
if which == "c2":
    n, k, b, var, snr, dt = 1 << 22, 1000, 1024, "dt2", "exact", torch.complex128
else:
    n, k, b, var, snr, dt = 1 << 24, 4096, 4096, "dt3", 20.0, torch.complex64
S = int(sys.argv[2]) if len(sys.argv) > 2 else 16
x, _ = make_batch(n, k, snr, S, dt, dev, chunk=4)
seeds = [case_seed(n, k, snr, i) for i in range(S)]
res = sfft_dt_batch(x, k, b, 4, 15, var, seeds=seeds)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for _ in range(2):
    res = sfft_dt_batch(x, k, b, 4, 15, var, seeds=seeds)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok", int(res.count.sum()))
