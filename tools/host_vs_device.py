"""Is a batched entry point bound by its host side?  For C1, C2, C3, C3', C4-DT3: the mean
CUDA-event time per call over back-to-back calls (what bench.py reports) beside the host's
own time to ISSUE one call (perf_counter around the call, stream drained first, no
synchronize after) — when the two agree, the GPU is waiting for the host."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from bench_suite import case_seed, make_batch  # noqa: E402
from paper_2011_05749_b200 import ffast_batch, plan_cycles, rffast_batch, sfft_dt_batch  # noqa: E402

dev = torch.device("cuda", 0)


def report(name, fn, reps=10):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    dev_ms = s.elapsed_time(e) / reps
    host = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        fn()
        host.append((time.perf_counter() - t) * 1e3)
    torch.cuda.synchronize()
    host.sort()
    print(f"{name}: events {dev_ms:.3f} ms per call, host issue median {host[len(host) // 2]:.3f} ms",
          flush=True)


which = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c1", "c2", "c3", "c4dt3"]
if "c1" in which:
    n, k = 124950, 40
    x, _ = make_batch(n, k, "exact", 8192, torch.complex128, dev, chunk=512)
    report("c1 (8192 signals)", lambda: ffast_batch(x, k, [49, 50, 51]))
    del x
if "c2" in which:
    n, k = 1 << 22, 1000
    x, _ = make_batch(n, k, "exact", 64, torch.complex128, dev, chunk=4)
    seeds = [case_seed(n, k, "exact", i) for i in range(64)]
    report("c2 (64 signals)", lambda: sfft_dt_batch(x, k, 1024, 4, 15, "dt2", seeds=seeds))
    del x
if "c3" in which:
    n, k, S = 511 * 512 * 513, 1000, 16
    x, _ = make_batch(n, k, 20.0, S, torch.complex128, dev, chunk=2)
    plans = [plan_cycles(n, k, "noisy", seed=case_seed(n, k, 20.0, i)) for i in range(S)]
    searches = [p[1] for p in plans]
    report("c3 literal (16 signals)", lambda: rffast_batch(x, k, [511, 512, 513], searches))
    f = list(plans[0][0].factors)
    report("c3 auto (16 signals)", lambda: rffast_batch(x, k, f, searches))
    del x
if "c4dt3" in which:
    n, k, S = 1 << 24, 4096, 32
    x, _ = make_batch(n, k, 20.0, S, torch.complex64, dev, chunk=4)
    seeds = [case_seed(n, k, 20.0, i) for i in range(S)]
    report("c4 dt3 (32 signals)", lambda: sfft_dt_batch(x, k, 4096, 4, 15, "dt3", seeds=seeds))
