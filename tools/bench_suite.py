#!/usr/bin/env python
"""Device throughput of every BASELINE config (bench.py reports config 5 as the headline).

    python tools/bench_suite.py [--configs c1,c2,c3,c3auto,c4dt3,c4dsfft] [--reps 3]

Inputs are resident in HBM before timing; times are CUDA events on the launching
stream, averaged over --reps after one warm-up.  Clean signals follow the
generate_test_case model (numpy-drawn truth, n * ifft on the device); for the
noisy configs the complex Gaussian noise at the configured SNR is drawn on the
device with torch's generator (same distribution as the reference's, not the
same stream — exact-input parity is the tests' job, not this timing run's).
Prints one JSON line per config.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
import zlib

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2011_05749_b200 import (  # noqa: E402
    DsfftConfig, ffast_batch, plan_cycles, rffast_batch, sfft_dt_batch,
)
from paper_2011_05749_b200.dsfft import dsfft_batch, dsfft_device  # noqa: E402
from paper_2011_05749_b200.signals import draw_truth  # noqa: E402


def case_seed(n, k, snr, trial):
    tag = "exact" if snr == "exact" else f"{float(snr):.9g}"
    return zlib.crc32(f"{n}|{k}|{tag}|0|{trial}".encode())


def make_batch(n, k, snr, batch, dtype, dev, chunk=4):
    x = torch.empty((batch, n), dtype=dtype, device=dev)
    truths = []
    for c0 in range(0, batch, chunk):
        c1 = min(batch, c0 + chunk)
        spec = torch.zeros((c1 - c0, n), dtype=torch.complex128, device=dev)
        for i in range(c0, c1):
            pos, coef = draw_truth(n, k, np.random.default_rng(case_seed(n, k, snr, i)))
            truths.append(set(pos.tolist()))
            spec[i - c0, torch.from_numpy(pos).to(dev)] = torch.from_numpy(coef).to(dev)
        sig = torch.fft.ifft(spec, dim=1) * n
        del spec
        if snr != "exact":
            p_sig = (sig.abs() ** 2).mean(dim=1, keepdim=True)
            std = torch.sqrt(p_sig / 10 ** (snr / 10) / 2)
            g = torch.Generator(device=dev).manual_seed(c0)
            sig = sig + std * torch.complex(torch.randn(sig.shape, device=dev, generator=g,
                                                        dtype=torch.float64),
                                            torch.randn(sig.shape, device=dev, generator=g,
                                                        dtype=torch.float64))
        x[c0:c1] = sig.to(dtype)
        del sig
    torch.cuda.synchronize()
    return x, truths


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps, (time.perf_counter() - t0) / reps


def recall(spectra_sets, truths):
    hits = sum(len(s & t) for s, t in zip(spectra_sets, truths))
    return hits / max(1, sum(len(t) for t in truths))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c3,c3auto,c4dt3,c4dsfft")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    todo = args.configs.split(",")

    def emit(name, batch, ms, wall, extra):
        line = {"config": name, "signals_per_launch": batch, "ms": ms,
                "signals_per_s": batch / (ms * 1e-3), "wall_ms": wall * 1e3}
        line.update(extra)
        print(json.dumps(line), flush=True)

    if "c1" in todo:
        n, k, f = 124950, 40, [49, 50, 51]
        x, tr = make_batch(n, k, "exact", 1024, torch.complex128, dev, chunk=256)
        one = x[:1].clone()
        # single-signal device latency: pre-allocated outputs, replayed as a CUDA graph
        r1 = ffast_batch(one, k, f)
        ws1 = torch.empty(1 << 20, dtype=torch.uint8, device=dev)
        ffast_batch(one, k, f, workspace=ws1, out=r1)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            ffast_batch(one, k, f, workspace=ws1, out=r1)
        ms1, wall1 = timed(g.replay, 50)
        ms, wall = timed(lambda: ffast_batch(x, k, f), args.reps)
        res = ffast_batch(x, k, f)
        emit("c1_ffast_n124950_k40", 1024, ms, wall,
             {"single_signal_us": ms1 * 1e3, "single_signal_wall_us": wall1 * 1e6,
              "recall": recall([set(res.spectrum(i).entries) for i in range(0, 1024, 64)],
                               tr[::64])})
        del x
    if "c2" in todo:
        n, k = 1 << 22, 1000
        x, tr = make_batch(n, k, "exact", 64, torch.complex128, dev, chunk=16)
        seeds = [case_seed(n, k, "exact", i) for i in range(64)]
        ms, wall = timed(lambda: sfft_dt_batch(x, k, 1024, 4, 15, "dt2", seeds=seeds), args.reps)
        res = sfft_dt_batch(x, k, 1024, 4, 15, "dt2", seeds=seeds)
        emit("c2_sfftdt2_n2^22_k1000_b1024", 64, ms, wall,
             {"recall": recall([set(res.spectrum(i).entries) for i in range(64)], tr)})
        del x
    if "c3" in todo or "c3auto" in todo:
        n, k = 511 * 512 * 513, 1000
        x, tr = make_batch(n, k, 20.0, 16, torch.complex128, dev, chunk=1)
        for name in ("c3", "c3auto"):
            if name not in todo:
                continue
            plan, search = plan_cycles(n, k, "noisy", seed=0)
            factors = [511, 512, 513] if name == "c3" else plan.factors
            ms, wall = timed(lambda: rffast_batch(x, k, factors, search), args.reps)
            res = rffast_batch(x, k, factors, search)
            emit(f"{name}_rffast_n134217216_k1000_20db_{'x'.join(map(str, factors))}", 16, ms,
                 wall, {"recall": recall([set(res.spectrum(i).entries) for i in range(16)], tr),
                        "rounds": res.rounds.tolist()})
        del x
    if "c4dt3" in todo or "c4dsfft" in todo:
        n, k = 1 << 24, 4096
        for snr in (10.0, 20.0, 30.0):
            x, tr = make_batch(n, k, snr, 32, torch.complex64, dev, chunk=4)
            if "c4dt3" in todo:
                seeds = [case_seed(n, k, snr, i) for i in range(32)]
                ms, wall = timed(lambda: sfft_dt_batch(x, k, 4096, 4, 15, "dt3", seeds=seeds),
                                 args.reps)
                res = sfft_dt_batch(x, k, 4096, 4, 15, "dt3", seeds=seeds)
                emit(f"c4_sfftdt3_n2^24_k4096_{int(snr)}db", 32, ms, wall,
                     {"recall": recall([set(res.spectrum(i).entries) for i in range(32)], tr)})
            if "c4dsfft" in todo:
                cfg = DsfftConfig(mode="noisy", seed=0, noise_std=float(np.sqrt(k * 10 ** (-snr / 10))))
                nsig = 4
                outs = []

                def run():
                    outs.clear()
                    for i in range(nsig):
                        outs.append(dsfft_device(x[i], k, cfg))

                ms, wall = timed(run, 1)
                emit(f"c4_dsfft_n2^24_k4096_{int(snr)}db", nsig, ms, wall,
                     {"recall": recall([set(o) for o in outs], tr[:nsig]), "mode": "sequential"})
                nb = 8
                batch_out = []

                def run_batch():
                    batch_out[:] = dsfft_batch(x[:nb], k, cfg, streams=8)

                ms, wall = timed(run_batch, 1)
                emit(f"c4_dsfft_n2^24_k4096_{int(snr)}db_batch8", nb, ms, wall,
                     {"recall": recall([set(o.entries) for o in batch_out], tr[:nb]),
                      "mode": "dsfft_batch, 8 streams"})
            del x
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
