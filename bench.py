#!/usr/bin/env python
"""Benchmark: FFAST sparse transforms/sec on BASELINE config 5 (the scaling config).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (N > 1; one rank per GPU)

Workload (BASELINE.json configs[4]): 8192 independent exactly-sparse signals,
complex64, N = 127*128*129 = 2,097,024, K = 256 unit-magnitude random-phase
tones, cycle plan 127/128/129 with delays 0,1,2 (explicit plan, SURVEY
Appendix A), sharded by signal across ranks (strong scaling: the 8192 total is
fixed) and the recovered [signals, K] slots all-gathered over NCCL.  One step =
one FFAST pass (|x|^2 stream for the exact thresholds, gather + 127/128/129-point
DFTs, GPU-resident peeling, top-K truncation, result gather) over the whole
resident batch.  Inputs are 137 GB >> 126 MB L2, so no L2 flush is needed.

Inputs follow generate_test_case's model (signals.py:81-117) with the bench's
per-signal seeds (bench.py:123-127): truth drawn on the host with numpy's
PCG64, the clean signal synthesised on the device (n * ifft, cast to c64).

--impl reference times the CPU restatement of the reference path (oracle/, a
numpy port pinned against the reference's outputs) on all host cores, on the
same workload, one bounded sample of signals per step.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
import zlib

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_SIG = 2097024
K = 256
FACTORS = [127, 128, 129]
TOTAL_SIGNALS = 8192
METRIC = "sparse transforms/sec (signals/s) at N,K; achieved HBM sector GB/s fraction"
UNIT = "signals/s"
SIGNAL_BYTES = N_SIG * 8  # complex64
# 32-byte sectors the gather touches per signal (unique per kernel), SURVEY §8d
GATHER_SECTOR_BYTES = None


def case_seed(n, k, snr, seed_base, trial):
    tag = "exact" if snr == "exact" else f"{float(snr):.9g}"
    return zlib.crc32(f"{n}|{k}|{tag}|{seed_base}|{trial}".encode()) ^ (seed_base << 1)


def gather_sector_bytes(n=N_SIG, factors=FACTORS, shifts=(0, 1, 2), esz=8):
    secs = set()
    for b in factors:
        j = np.arange(b, dtype=np.int64) * (n // b)
        for t in shifts:
            secs.update(((j - t) % n * esz // 32).tolist())
    return 32 * len(secs)


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self.proc = None
        time.sleep(0.15)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- inputs


def synth_signals(x, first_trial: int, dev, chunk: int = 32):
    """Fill x[i] with trial first_trial+i of config 5 (n*ifft of the sparse truth, c64)."""
    import torch

    from paper_2011_05749_b200.signals import draw_truth

    count = x.shape[0]
    spec = torch.zeros((chunk, N_SIG), dtype=torch.complex128, device=dev)
    truths = []
    for c0 in range(0, count, chunk):
        c1 = min(count, c0 + chunk)
        spec.zero_()
        for i in range(c0, c1):
            rng = np.random.default_rng(case_seed(N_SIG, K, "exact", 0, first_trial + i))
            pos, coef = draw_truth(N_SIG, K, rng)
            truths.append((pos, coef))
            spec[i - c0, torch.from_numpy(pos).to(dev)] = torch.from_numpy(coef).to(dev)
        x[c0:c1] = (torch.fft.ifft(spec[: c1 - c0], dim=1) * N_SIG).to(torch.complex64)
    del spec
    return truths


# ----------------------------------------------------------------------------- our arm


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2011_05749_b200 import _lib
    from paper_2011_05749_b200.batch import ffast_batch, ffast_workspace_bytes

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    from paper_2011_05749_b200.shard import gather_slots, max_over_ranks, shard_range

    total = args.signals
    first, stop = shard_range(total, rank, world)
    per = stop - first
    if total % world:
        raise SystemExit("--signals must be a multiple of the rank count (equal result slots)")

    x = torch.empty((per, N_SIG), dtype=torch.complex64, device=dev)
    truths = synth_signals(x, first, dev)
    torch.cuda.synchronize()

    lib = _lib.load()  # noqa: F841  (fail loudly here if the library is missing)
    code = _lib.AFFT_C64
    ws = torch.empty(ffast_workspace_bytes(N_SIG, code, per, FACTORS), dtype=torch.uint8,
                     device=dev)
    res = ffast_batch(x, K, FACTORS, workspace=ws)
    stream = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]

    def step(i=None):
        """One FFAST pass over the resident batch: a single afft_ffast call (one
        ffast_fused_kernel launch), then the NCCL gather of the result slots."""
        if i is not None:
            ev[i][0].record(stream)
        ffast_batch(x, K, FACTORS, workspace=ws, out=res)
        if i is not None:
            ev[i][1].record(stream)
        if world > 1:
            gather_slots(res.pos, res.val, res.count)

    # afft_ffast's default for this batch: one ffast_fused_kernel launch (>= 40 signals
    # per SM) or one ffast_parts_kernel launch (split streams, smaller per-rank batches)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    fused = per >= 40 * sms
    kernel_name = "ffast_fused_kernel" if fused else "ffast_parts_kernel"
    launches_per_step = 1

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # correctness of the measured pass: every recovered tone is a true tone
    cnt = res.count.cpu().numpy()
    pos = res.pos.cpu().numpy()
    exact = sum(int(cnt[i]) == K and set(pos[i, :K].tolist()) == set(truths[i][0].tolist())
                for i in range(per))
    kept = sum(int(c) for c in cnt)
    true_kept = sum(len(set(pos[i, :int(cnt[i])].tolist()) & set(truths[i][0].tolist()))
                    for i in range(per))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        start.record(stream)
        for i in range(args.steps):
            step(i)
        end.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = start.elapsed_time(end)
    kern_ms = statistics.mean(a.elapsed_time(b) for a, b in ev)
    ms, kern_ms = max_over_ranks([ms, kern_ms], dev)
    ms_per_step = ms / args.steps

    # the two-stream pipelined alternative (afft_ffast mode 2) for comparison
    os.environ["AFFT_FFAST_MODE"] = "2"
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    step()
    e0.record(stream)
    for _ in range(3):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    fused_ms = e0.elapsed_time(e1) / 3
    del os.environ["AFFT_FFAST_MODE"]

    # e2e on every rank at once (each GPU has its own PCIe link): whole-job signals over
    # the slowest rank's time
    if world > 1:
        dist.barrier()
    e2e = run_e2e(args, dev, x, world)
    e2e_ms, copy_ms = max_over_ranks([e2e["ms_per_step"], e2e.pop("_copy_ms")], dev)
    e2e.update({"value": world * e2e["signals_per_step"] / (e2e_ms * 1e-3),
                "ms_per_step": e2e_ms, "signals_per_step": world * e2e["signals_per_step"],
                "h2d_bytes_per_step": world * e2e["h2d_bytes_per_step"],
                "d2h_bytes_per_step": world * e2e["d2h_bytes_per_step"],
                "frac_of_h2d_bound": copy_ms / e2e_ms, "ranks": world})
    read_gbs = read_stream_gbs(x, dev) if rank == 0 else None
    context = dense_fft_context(x, dev) if rank == 0 else None
    cpu = cpu_baseline_sample(x[: args.cpu_signals]) if (rank == 0 and world == 1) else None

    if rank == 0:
        peak, peak_src = load_peaks()
        gsec = gather_sector_bytes()
        alg_bytes = per * (SIGNAL_BYTES + gsec)
        achieved = alg_bytes / (kern_ms * 1e-3) / 1e9
        traffic = None
        prof = os.path.join(ROOT, "profiles", "ncu_ffast_fused_traffic.json")
        if os.path.exists(prof):
            with open(prof) as fh:
                d = json.load(fh)
            traffic = float(d["dram_bytes_per_signal"]) * per
        value = total / (ms_per_step * 1e-3)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "c64 in, f64 compute", "data": "synthetic (generate_test_case model, seeded)",
            "config": {
                "workload": "config5_ffast_n2097024_k256_127x128x129_c64",
                "n": N_SIG, "k": K, "factors": FACTORS, "shifts": [0, 1, 2],
                "signals_total": total, "signals_per_rank": per,
                "l2": "inputs 137 GB >> 126 MB L2 (no flush needed)",
                "parallelism": f"signal-sharded x{world}, NCCL all-gather of result slots",
                "exact_recovered_fraction": exact / per, "true_tone_fraction": true_kept / max(1, kept),
                "step_kernels_ms": kern_ms,
                "step": ("one ffast_fused_kernel launch per step (afft_ffast mode 0): each CTA "
                         "gathers + transforms its signal, streams its |x|^2, then peels it"
                         if fused else
                         "one ffast_parts_kernel launch per step (afft_ffast mode 4): several "
                         "CTAs stream parts of each signal's |x|^2, the last one decodes it"),
                "pipelined_two_stream_ms": fused_ms,
            },
            "roofline": {
                "kernel": f"{kernel_name} (|x|^2 stream + gather/DFT + peel + truncate)",
                "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "peak_source": peak_src,
                "algorithmic_bytes_per_launch": alg_bytes, "traffic": traffic,
                "algorithmic_bytes_per_signal": SIGNAL_BYTES + gsec,
                "gather_sector_bytes_per_signal": gsec,
                # the copy peak counts read+write bytes; this kernel only reads, and a
                # pure read stream runs faster than a copy on HBM3e.  Measured live: the
                # library's |x|^2 stream alone over the same resident batch.
                "read_stream_gbs_live": read_gbs,
                "frac_of_read_stream": achieved / read_gbs if read_gbs else None,
            },
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
            "context": context,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_e2e(args, dev, x, world):
    """Same metric through the public API with HOST (pinned) buffers: H2D of every
    step's signals + the decode + D2H of the result slots, all timed.  Per rank; the
    caller combines the ranks (max time)."""
    import torch

    from paper_2011_05749_b200.batch import ffast_batch

    m = min(args.e2e_signals, x.shape[0])
    host = torch.empty((m, N_SIG), dtype=torch.complex64, pin_memory=True)
    host.copy_(x[:m])
    dbuf = torch.empty((m, N_SIG), dtype=torch.complex64, device=dev)
    res = ffast_batch(dbuf.copy_(host, non_blocking=True), K, FACTORS)
    hpos = torch.empty((m, K), dtype=torch.int64, pin_memory=True)
    hval = torch.empty((m, K), dtype=torch.complex128, pin_memory=True)
    hcnt = torch.empty(m, dtype=torch.int32, pin_memory=True)
    stream = torch.cuda.current_stream()

    def step():
        dbuf.copy_(host, non_blocking=True)
        ffast_batch(dbuf, K, FACTORS, out=res)
        hpos.copy_(res.pos, non_blocking=True)
        hval.copy_(res.val, non_blocking=True)
        hcnt.copy_(res.count, non_blocking=True)

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    steps = max(2, min(args.steps, 5))
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    for _ in range(steps):
        step()
    e.record(stream)
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / steps
    # the bound: the same pinned H2D copy alone (PCIe)
    s.record(stream)
    for _ in range(steps):
        dbuf.copy_(host, non_blocking=True)
    e.record(stream)
    torch.cuda.synchronize()
    copy_ms = s.elapsed_time(e) / steps
    return {"value": m / (ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": m * SIGNAL_BYTES,
            "d2h_bytes_per_step": m * K * (8 + 16) + m * 4, "signals_per_step": m,
            "ms_per_step": ms, "api": "paper_2011_05749_b200.ffast_batch (afft_ffast) on pinned host",
            "h2d_alone_gbs": m * SIGNAL_BYTES / copy_ms / 1e6,
            "frac_of_h2d_bound": copy_ms / ms, "_copy_ms": copy_ms}


def read_stream_gbs(x, dev, reps: int = 3):
    """Read-only HBM bandwidth over the resident batch: afft_sumsq (one pass over
    every signal, partial sums out) timed with CUDA events on the launching stream."""
    import torch

    from paper_2011_05749_b200 import _lib

    lib = _lib.load()
    S = int(x.shape[0])
    nparts = int(lib.afft_sumsq_parts(N_SIG, _lib.AFFT_C64))
    part = torch.empty((S, nparts), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream

    def once():
        _lib.check(lib.afft_sumsq(x.data_ptr(), _lib.AFFT_C64, N_SIG, S, N_SIG,
                                  part.data_ptr(), sp), "sumsq")

    once()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(stream)
    for _ in range(reps):
        once()
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    return S * SIGNAL_BYTES / (ms * 1e-3) / 1e9


def dense_fft_context(x, dev):
    """Context only (north_star): a dense full-length FFT of the same N — cuFFT on this
    B200 (via torch, c64) and numpy on one host core — in signals/s."""
    import torch

    m = min(512, x.shape[0])
    xs = x[:m]
    out = torch.empty_like(xs)

    def run():
        out.copy_(torch.fft.fft(xs, dim=1))

    run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        run()
    b.record()
    torch.cuda.synchronize()
    gpu_ms = a.elapsed_time(b) / 3
    # the same transform in float64 arithmetic: cuFFT c128 and this library's
    # four-step K2' (afft_bucketize with b = N, tau = 0 — y = fft(x) / N)
    from paper_2011_05749_b200 import _device, _lib

    m2 = min(64, x.shape[0])
    x2 = x[:m2]
    x2c = x2.to(torch.complex128)
    out2 = torch.empty((m2, N_SIG), dtype=torch.complex128, device=dev)
    lib = _lib.load()
    sb, ns = _lib.host_i64([0])

    def run_c128():
        out2.copy_(torch.fft.fft(x2c, dim=1))

    def run_ours():
        _lib.check(lib.afft_bucketize(x2.data_ptr(), _device.dtype_code(x2), N_SIG, m2, N_SIG, N_SIG,
                                      sb, ns, out2.data_ptr(), N_SIG, N_SIG, 1,
                                      _device.stream_ptr()), "bucketize(b=N)")

    def timed(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    c128_ms = timed(run_c128)
    ours_ms = timed(run_ours)
    del x2c, out2
    host = x[0].cpu().numpy()
    t0 = time.perf_counter()
    for _ in range(3):
        np.fft.fft(host.astype(np.complex128))
    cpu_s = (time.perf_counter() - t0) / 3
    return {"dense_fft_gpu_signals_per_s": m / (gpu_ms * 1e-3), "dense_fft_gpu": "cuFFT c64 (torch.fft)",
            "dense_fft_gpu_c128_signals_per_s": m2 / (c128_ms * 1e-3),
            "dense_fft_ours_signals_per_s": m2 / (ours_ms * 1e-3),
            "dense_fft_ours": "four-step K2' (afft_bucketize, b = N), c64 in, f64 compute, c128 out",
            "dense_fft_cpu_signals_per_s": 1.0 / cpu_s, "dense_fft_cpu": "numpy pocketfft c128, 1 core",
            "note": "context only; not part of the measured path"}


def cpu_baseline_sample(xs):
    """The oracle port timed on one host core over a bounded sample of the same signals."""
    from oracle import ffast as oracle_ffast

    arr = xs.cpu().numpy()
    t0 = time.perf_counter()
    done = 0
    for row in arr:
        oracle_ffast.ffast(row.astype(np.complex128), K, FACTORS)
        done += 1
        if time.perf_counter() - t0 > 20.0:
            break
    dt = time.perf_counter() - t0
    return {"value": done / dt, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"{done} config-5 signals (same device-synthesised inputs), oracle/ffast.py, "
                      "1 thread, upcast c64->c128 as the reference does"}


# ----------------------------------------------------------------------------- reference arm


def _ref_worker(args_tuple):
    wid, per_step, steps, warmup, barrier, q = args_tuple
    from oracle import ffast as oracle_ffast
    from paper_2011_05749_b200.signals import generate_test_case

    xs = []
    for j in range(per_step):
        seed = case_seed(N_SIG, K, "exact", 0, wid * per_step + j)
        xs.append(generate_test_case(N_SIG, K, "exact", seed).signal.astype(np.complex64)
                  .astype(np.complex128))
    for _ in range(warmup):
        oracle_ffast.ffast(xs[0], K, FACTORS)
    times = []
    for _ in range(steps):
        barrier.wait()
        t0 = time.perf_counter()
        for x in xs:
            oracle_ffast.ffast(x, K, FACTORS)
        times.append((t0, time.perf_counter()))
    q.put(times)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    import multiprocessing as mp

    # one BLAS / OpenMP thread per worker process, fixed before the workers import numpy
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"
    cores = os.cpu_count() or 1
    per_step = 4  # signals per core per step: amortises the per-step barrier
    ctx = mp.get_context("spawn")
    barrier = ctx.Barrier(cores)
    q = ctx.Queue()
    procs = [ctx.Process(target=_ref_worker,
                         args=((w, per_step, args.steps, args.warmup, barrier, q),))
             for w in range(cores)]
    for p in procs:
        p.start()
    results = [q.get() for _ in procs]
    for p in procs:
        p.join()
    step_ms = []
    for s in range(args.steps):
        t0 = min(r[s][0] for r in results)
        t1 = max(r[s][1] for r in results)
        step_ms.append((t1 - t0) * 1e3)
    ms = statistics.mean(step_ms)
    value = cores * per_step / (ms * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "c128 (reference upcasts c64)",
        "data": "synthetic (generate_test_case, seeded)", "impl": "reference",
        "config": {"workload": "config5_ffast_n2097024_k256_127x128x129_c64", "n": N_SIG, "k": K,
                   "factors": FACTORS, "signals_per_step": cores * per_step},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{cores * per_step} signals per step ({per_step} per core), "
                                   "oracle/ffast.py numpy port of the reference FFAST path, "
                                   "signal generation excluded as bench.py:172-176 does"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--signals", type=int, default=TOTAL_SIGNALS)
    ap.add_argument("--e2e-signals", type=int, default=256)
    ap.add_argument("--cpu-signals", type=int, default=128)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
