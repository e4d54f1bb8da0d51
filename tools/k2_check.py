"""K2' large-b bucketization: accuracy against torch.fft (c128) and timing, for the
register-resident pass (default) or the smem Stockham pass (AFFT_FFT_SMEM=1)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2011_05749_b200.bucketize import bucketize_device  # noqa: E402

dev = torch.device("cuda", 0)
n = 1 << 24
g = torch.Generator(device=dev).manual_seed(0)
x64 = torch.randn(n, dtype=torch.complex64, device=dev, generator=g)
x128 = x64.to(torch.complex128)
mode = "smem" if os.environ.get("AFFT_FFT_SMEM") == "1" else "reg"
for lg in [int(a) for a in sys.argv[1:]] or [13, 14, 16, 17, 20, 22, 23, 24]:
    b = 1 << lg
    L = n // b
    shifts = list(range(min(L, 8)))
    for x, name in ((x64, "c64"), (x128, "c128")):
        out = bucketize_device(x, b, shifts)
        idx = torch.arange(b, device=dev) * L
        err = 0.0
        for t, tau in enumerate(shifts):
            ref = torch.fft.fft(x128[(idx - tau) % n]) / b
            got = out[t] if out.dim() == 2 else out
            err = max(err, float((got - ref).abs().max() / ref.abs().max()))
        torch.cuda.synchronize()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            bucketize_device(x, b, shifts)
        e.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(e) / 5
        pts = len(shifts) * b
        print(f"{mode} {name} b=2^{lg} shifts={len(shifts)} {ms:.3f} ms ({pts / ms / 1e6:.0f} "
              f"Gpts/s) rel err {err:.2e}", flush=True)
