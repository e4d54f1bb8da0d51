"""Four-step bucketization timing at DSFFT-like sizes (diagnostic): n = 2^24 c64,
b = 2^k for the deepest layers, U cosets = n / b (every residue)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2011_05749_b200.bucketize import bucketize_device  # noqa: E402

dev = torch.device("cuda", 0)
n = 1 << 24
x = torch.randn(n, dtype=torch.complex64, device=dev)
only = [int(a) for a in sys.argv[1:]] or [13, 16, 20, 22, 23, 24]
for lg in only:
    b = 1 << lg
    L = n // b
    shifts = list(range(min(L, 8)))
    bucketize_device(x, b, shifts)
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        bucketize_device(x, b, shifts)
    e.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(e) / 5
    pts = len(shifts) * b
    print(f"b=2^{lg} shifts={len(shifts)} {ms:.3f} ms  ({pts / ms / 1e6:.1f} Gpts/s; "
          f"out {pts * 16 / ms / 1e6:.0f} GB/s)", flush=True)
