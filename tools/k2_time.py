"""Time the K2' dense transform (b = n, tau = 0) at n = 2^24 (c64 and c128 input) and
n = 2^22 x 4 shifts with CUDA events; prints ms per call, the effective algorithmic
bandwidth of the passes, and a digest of the output so runs with AFFT_FFT_TMA=0/1
can be compared bit for bit.

    AFFT_FFT_TMA=1 python tools/k2_time.py
"""
import hashlib
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_05749_b200.bucketize import bucketize_device  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(7)
out = {"tma": os.environ.get("AFFT_FFT_TMA", "1")}
for name, n, dt in (("2^24 c64", 1 << 24, torch.complex64), ("2^24 c128", 1 << 24, torch.complex128)):
    x = torch.randn(n, dtype=torch.complex128, device=dev, generator=g).to(dt)
    y = bucketize_device(x, n, [0])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        y = bucketize_device(x, n, [0])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    esz = 8 if dt == torch.complex64 else 16
    alg = n * esz + n * 16 + 2 * 2 * n * 16  # pass 1 reads x, writes c128; passes 2, 3 r+w
    out[name] = {"ms": ms, "alg_gbs": alg / ms / 1e6,
                 "digest": hashlib.sha256(y.cpu().numpy().tobytes()).hexdigest()[:16]}
print(json.dumps(out))
