"""Small, ncu-friendly driver of the bench kernel: config-5 FFAST over a few signals.

    python tools/ncu_target.py [--signals 296] [--iters 3]

Run it plain first, then under ncu (see profiles/README.md for the exact commands).
"""

import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2011_05749_b200 import ffast_batch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--signals", type=int, default=296)
    ap.add_argument("--iters", type=int, default=3)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    x = torch.empty((args.signals, bench.N_SIG), dtype=torch.complex64, device=dev)
    bench.synth_signals(x, 0, dev)
    res = ffast_batch(x, bench.K, bench.FACTORS)
    for _ in range(args.iters):
        ffast_batch(x, bench.K, bench.FACTORS, out=res)
    torch.cuda.synchronize()
    print("ok", int(res.count.sum()))


if __name__ == "__main__":
    main()
