"""Run the CSV experiment grid (paper_2011_05749_b200.experiments) on the GPU.

    python tools/run_grid.py [--out profiles/r01_grid.csv] [--trials 2]

Default grid: every algorithm at small power-of-two and co-prime sizes, exact and
20 dB — the shape of the reference's own sweeps, small enough for a minute.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2011_05749_b200.experiments import ALGORITHMS, ExperimentConfig, run_suite  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/grid.csv")
    ap.add_argument("--trials", type=int, default=2)
    ap.add_argument("--n", default="4095,4096,65535,65536,1048575,1048576")
    ap.add_argument("--k", default="4,16")
    ap.add_argument("--snr", default="exact,20")
    args = ap.parse_args()
    snrs = [s if s == "exact" else float(s) for s in args.snr.split(",")]
    cfg = ExperimentConfig(list(ALGORITHMS), [int(v) for v in args.n.split(",")],
                           [int(v) for v in args.k.split(",")], snrs, trials=args.trials,
                           out_path=args.out)
    rows = run_suite(cfg)
    print(f"{len(rows)} rows -> {args.out}")


if __name__ == "__main__":
    main()
