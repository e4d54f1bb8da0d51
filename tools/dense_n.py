"""Dense K2' transforms of N = 2,097,024 = 127 x 128 x 129 (config 5's size; b = n,
tau = 0), c64 in (diagnostic, for ncu): python tools/dense_n.py [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_05749_b200.bucketize import bucketize_device  # noqa: E402

dev = torch.device("cuda", 0)
n = 127 * 128 * 129
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
x = torch.randn(n, dtype=torch.complex64, device=dev)
for _ in range(reps):
    y = bucketize_device(x, n, [0])
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    bucketize_device(x, n, [0])
e1.record()
torch.cuda.synchronize()
ref = torch.fft.fft(x.to(torch.complex128)) / n
print("ms", e0.elapsed_time(e1) / 20, "rel err", float((y.reshape(-1) - ref).abs().max() / ref.abs().max()))
