"""Config-5 step time, fused kernel (mode 0) vs split streams (mode 4, `parts` CTAs per
signal), at the per-rank batch sizes of the scaling run (diagnostic)."""
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
for S in [int(v) for v in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["8192", "2048", "1024"])]:
    xs = x[:S]
    res = ffast_batch(xs, bench.K, bench.FACTORS)
    ref = None
    row = {}
    for mode, parts in (("0", None), ("1", None), ("4", "2"), ("4", "3"), ("4", "4"), ("4", "6"), ("4", "8"), ("4", "12")):
        os.environ["AFFT_FFAST_MODE"] = mode
        if parts:
            os.environ["AFFT_FFAST_PARTS"] = parts
        ms = t(lambda: ffast_batch(xs, bench.K, bench.FACTORS, out=res), reps=10)
        got = (res.count.clone(), res.pos.clone())
        ref = ref or got
        assert torch.equal(ref[0], got[0]) and torch.equal(ref[1], got[1]), (mode, parts)
        row[f"m{mode}" + (f"p{parts}" if parts else "")] = round(ms, 3)
    print(S, row, flush=True)
