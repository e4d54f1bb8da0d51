"""Config-5 step time vs signals per GPU (what each rank sees under the strong-scaling
bench at N = 1/2/4/8: 8192/4096/2048/1024 signals), fused kernel, CUDA events."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import bench  # noqa: E402
from ffast_modes import t  # noqa: E402
from paper_2011_05749_b200 import ffast_batch  # noqa: E402

dev = torch.device("cuda", 0)
x = torch.empty((8192, bench.N_SIG), dtype=torch.complex64, device=dev)
bench.synth_signals(x, 0, dev)
base = None
for S in (8192, 4096, 3072, 2048, 1536, 1024, 512, 296):
    xs = x[:S]
    res = ffast_batch(xs, bench.K, bench.FACTORS)
    row = {}
    for mode in ("0", "1", "auto"):
        if mode == "auto":
            os.environ.pop("AFFT_FFAST_MODE", None)
        else:
            os.environ["AFFT_FFAST_MODE"] = mode
        row[mode] = t(lambda: ffast_batch(xs, bench.K, bench.FACTORS, out=res), reps=10)
    rate = S / row["auto"] * 1e3
    base = base or rate
    print(f"signals {S:5d}: fused {row['0']:7.3f} ms, pre-pass {row['1']:7.3f} ms, default "
          f"{row['auto']:7.3f} ms = {rate:9.0f} signals/s ({rate / base:.3f} of the 8192 rate)",
          flush=True)
