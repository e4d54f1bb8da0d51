"""Host share of the batched entry points (diagnostic): per config, the bench's CUDA-event
time per call with the per-signal seeds (host draws every signal's random shifts, as
bench.py does), the same with the shifts drawn beforehand, and the host time of the
draws alone; DSFFT per-signal streams vs lockstep through dsfft_batch.
    python tools/host_share.py"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import _timed, case_seed, synth_batch  # noqa: E402
from paper_2011_05749_b200 import DsfftConfig, dsfft_batch, sfft_dt_batch  # noqa: E402
from paper_2011_05749_b200.oneshot import OneShotConfig, random_shifts  # noqa: E402

dev = torch.device("cuda", 0)
out = {}
for name, n, k, S, b, var, dt, snr in (("c2", 1 << 22, 1000, 64, 1024, "dt2", torch.complex128, "exact"),
                                       ("c4dt3", 1 << 24, 4096, 32, 4096, "dt3", torch.complex64, 20.0)):
    x, _ = synth_batch(n, k, snr, list(range(S)), dt, dev, chunk=4)
    seeds = [case_seed(n, k, snr, 0, i) for i in range(S)]
    t = time.perf_counter()
    rs = [random_shifts(n, OneShotConfig(b=b, a_m=4, p=15, seed=int(s))) for s in seeds]
    host_ms = (time.perf_counter() - t) * 1e3
    with_seeds = _timed(lambda: sfft_dt_batch(x, k, b, 4, 15, var, seeds=seeds), 20)
    pre = _timed(lambda: sfft_dt_batch(x, k, b, 4, 15, var, rand_shifts=rs), 20)
    out[name] = {"signals": S, "ms_with_seeds": with_seeds, "ms_shifts_drawn_before": pre,
                 "host_draw_ms": host_ms}
    if name == "c4dt3":
        cfgs = [DsfftConfig(mode="noisy", seed=s, noise_std=float(np.sqrt(k * 10 ** (-snr / 10))))
                for s in seeds]
        out["c4dsfft"] = {
            "per_signal_ms": _timed(lambda: dsfft_batch(x, k, cfgs), 3),
            "lockstep_ms": _timed(lambda: dsfft_batch(x, k, cfgs, lockstep=True), 3),
            "lockstep_4x8_ms": _timed(lambda: dsfft_batch(x, k, cfgs, lockstep=True, streams=4), 3),
            "lockstep_2x16_ms": _timed(lambda: dsfft_batch(x, k, cfgs, lockstep=True, streams=2, chunk=16), 3),
        }
    del x
    torch.cuda.empty_cache()
print(json.dumps(out))
