"""The 2^24-point K2' transform (b = n) against cuFFT c128 (relative max error) and its
time per call with CUDA events — run with AFFT_FFT_4K=0 (three radix-256 passes) and
=1 (two radix-4096 passes, the default) to compare.   python tools/k4_check.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_05749_b200.bucketize import bucketize_device  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(7)
out = {"fft4k": os.environ.get("AFFT_FFT_4K", "1")}
n = 1 << 24
for name, dt in (("c64", torch.complex64), ("c128", torch.complex128)):
    x = torch.randn(n, dtype=torch.complex128, device=dev, generator=g).to(dt)
    y = bucketize_device(x, n, [0]).reshape(-1)
    ref = torch.fft.fft(x.to(torch.complex128)) / n
    err = float((y - ref).abs().max() / ref.abs().max())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        bucketize_device(x, n, [0])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    out[name] = {"ms": ms, "rel_max_err_vs_cufft": err}
print(json.dumps(out))
