"""Config-1 batched FFAST (n = 124,950, k = 40, c128) under each afft_ffast mode and
batch size (diagnostic): the mode rule was tuned on config 5's 16.8 MB signals."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from bench_suite import make_batch  # noqa: E402
from ffast_modes import t  # noqa: E402
from paper_2011_05749_b200 import ffast_batch  # noqa: E402

n, k, f = 49 * 50 * 51, 40, [49, 50, 51]
dev = torch.device("cuda", 0)
x, _ = make_batch(n, k, "exact", 8192, torch.complex128, dev, chunk=512)
for S in (1024, 4096, 8192):
    xs = x[:S]
    res = ffast_batch(xs, k, f)
    row = {}
    for mode in ("0", "1", "2"):
        os.environ["AFFT_FFAST_MODE"] = mode
        row[mode] = t(lambda: ffast_batch(xs, k, f, out=res), reps=10)
    os.environ.pop("AFFT_FFAST_MODE")
    best = min(row, key=row.get)
    print(f"signals {S}: " + ", ".join(f"mode {m} {v:.3f} ms ({S / v * 1e3 / 1e6:.2f} M/s)"
                                      for m, v in row.items()) + f"; best {best}", flush=True)
