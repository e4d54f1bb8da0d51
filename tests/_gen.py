"""Parallel host generation of golden inputs (test infrastructure).

The config-sized parity tests need the exact host inputs the reference decoded
(generate_test_case is bit-identical to the reference's, sha256-pinned in
test_oracle_golden.py).  At N = 2^24 or 134M one signal takes 3-35 s of numpy on
one core, so signals are produced by a spawn-context process pool and streamed
back in order.
"""

from __future__ import annotations

import os


def _one(args):
    n, k, snr, seed, c64 = args
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ.setdefault(var, "1")
    import numpy as np

    from paper_2011_05749_b200.signals import generate_test_case

    x = generate_test_case(n, k, snr, seed).signal
    return x.astype(np.complex64) if c64 else x


def signals(specs, workers: int | None = None, gb_per_worker: float = 1.0):
    """Yield generate_test_case(n, k, snr, seed).signal (c64 if asked) for each spec
    (n, k, snr, seed, c64), in order."""
    import multiprocessing as mp

    cores = os.cpu_count() or 1
    w = workers or cores
    try:
        import psutil

        w = max(1, min(w, int(0.6 * psutil.virtual_memory().available / 2**30 / gb_per_worker)))
    except Exception:
        pass
    w = max(1, min(w, len(specs)))
    if w == 1:
        for s in specs:
            yield _one(s)
        return
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ.setdefault(var, "1")
    ctx = mp.get_context("spawn")
    with ctx.Pool(w) as pool:
        yield from pool.imap(_one, specs, chunksize=1)
