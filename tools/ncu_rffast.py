"""Small driver of the config-3 R-FFAST path for launch lists / ncu (diagnostic)."""

import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from bench_suite import make_batch  # noqa: E402
from paper_2011_05749_b200 import plan_cycles, rffast_batch  # noqa: E402

n, k = 511 * 512 * 513, 1000
signals = int(sys.argv[1]) if len(sys.argv) > 1 else 4
auto = len(sys.argv) > 2 and sys.argv[2] == "auto"
x, _ = make_batch(n, k, 20.0, signals, torch.complex128, torch.device("cuda", 0), chunk=1)
plan, search = plan_cycles(n, k, "noisy", seed=0)
factors = plan.factors if auto else [511, 512, 513]
res = rffast_batch(x, k, factors, search)
torch.cuda.synchronize()
print("rounds", res.rounds.tolist())
