#!/usr/bin/env python
"""Benchmark: sparse transforms/sec on the BASELINE configs (config 5 is the headline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

With --gpus N > 1 and no torchrun environment, bench.py re-launches itself under
`python -m torch.distributed.run --nproc-per-node N` (one rank per GPU, NCCL); under
torchrun it checks WORLD_SIZE == N.

Headline workload (BASELINE.json configs[4], the scaling config): 8192 independent
exactly-sparse signals, complex64, N = 127*128*129 = 2,097,024, K = 256
unit-magnitude random-phase tones, cycle plan 127/128/129 with delays 0,1,2
(explicit plan), sharded by signal across ranks (strong
scaling: the 8192 total is fixed) and the recovered [signals, K] slots
all-gathered over NCCL.  One step = one FFAST pass (|x|^2 stream for the exact
thresholds, gather + 127/128/129-point DFTs, GPU-resident peeling, top-K
truncation, result gather) over the whole resident batch.  Inputs are 137 GB >>
126 MB L2, so no L2 flush is needed.

At N = 1 the line also carries `configs`: configs 1-4 (C1, C2, C3 with the literal
and the auto plan, C4 sFFT-DT3 and C4 DSFFT at 10/20/30 dB) timed on the same GPU
through their batched entry points, each with its roofline and the reference
package's own CPU time (baseline/_ref, SURVEY Appendix A calls).

Inputs follow generate_test_case's model (signals.py:81-117) with the reference
bench's per-signal seeds (bench.py:123-127): truth drawn on the host with numpy's
PCG64, the clean signal synthesised on the device (n * ifft); for the noisy
configs the Gaussian noise at the stated SNR is drawn on the device (same
distribution as the reference's, not numpy's stream: exact-input parity is the
tests' job, tests/test_gpu_parity_batch.py).

--impl reference times the reference package itself (baseline/_ref, installed
from /root/reference) on all host cores, on the headline workload.
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
REF_DIR = os.path.join(ROOT, "baseline", "_ref")

N_SIG = 2097024
K = 256
FACTORS = [127, 128, 129]
TOTAL_SIGNALS = 8192
METRIC = "sparse transforms/sec (signals/s) at N,K; achieved HBM sector GB/s fraction"
UNIT = "signals/s"
SIGNAL_BYTES = N_SIG * 8  # complex64
WORKLOAD = "config5_ffast_n2097024_k256_127x128x129_c64"


def case_seed(n, k, snr, seed_base, trial):
    """The reference bench's per-cell seed (bench.py:123-127)."""
    tag = "exact" if snr == "exact" else f"{float(snr):.9g}"
    return zlib.crc32(f"{n}|{k}|{tag}|{seed_base}|{trial}".encode()) ^ (seed_base << 1)


def gather_sector_bytes(n=N_SIG, factors=FACTORS, shifts=(0, 1, 2), esz=8):
    """Unique 32-byte sectors the gather touches per signal (SURVEY §8d accounting)."""
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


def load_fp64_peak():
    path = os.path.join(ROOT, "profiles", "r01_fp64_peak.json")
    with open(path) as fh:
        d = json.load(fh)
    return float(d["fp64_dfma_tflops"]), "measured DFMA probe (tools/fp64_peak.cu, profiles/r01_fp64_peak.json)"


def load_json(name):
    path = os.path.join(ROOT, "profiles", name)
    if not os.path.exists(path):
        return None
    with open(path) as fh:
        return json.load(fh)


def host_info():
    info = {"cores": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        keep = ("Model name", "Socket(s)", "Core(s) per socket", "Thread(s) per core", "CPU(s)")
        info["lscpu"] = {ln.split(":", 1)[0].strip(): ln.split(":", 1)[1].strip()
                         for ln in out.splitlines()
                         if ":" in ln and ln.split(":", 1)[0].strip() in keep}
    except Exception:
        pass
    try:
        import psutil

        info["ram_gb"] = round(psutil.virtual_memory().total / 2**30, 1)
    except Exception:
        pass
    return info


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


# ============================================================================ the reference
#
# The reference package itself (baseline/_ref, pip-installed from /root/reference),
# called exactly as SURVEY Appendix A maps each BASELINE config to its public API.

REF_CONFIGS = {
    "c1": {"n": 124950, "k": 40, "snr": "exact", "c64": False},
    "c2": {"n": 1 << 22, "k": 1000, "snr": "exact", "c64": False},
    "c3": {"n": 511 * 512 * 513, "k": 1000, "snr": 20.0, "c64": False},
    "c3auto": {"n": 511 * 512 * 513, "k": 1000, "snr": 20.0, "c64": False},
    "c4dt3": {"n": 1 << 24, "k": 4096, "snr": 20.0, "c64": True},
    "c4dsfft": {"n": 1 << 24, "k": 4096, "snr": 20.0, "c64": True},
    "c5": {"n": N_SIG, "k": K, "snr": "exact", "c64": True},
}
# host RAM one reference call needs (generation + the call), to bound the process pool
REF_GB_PER_PROC = {"c1": 0.2, "c2": 1.0, "c3": 12.0, "c3auto": 12.0, "c4dt3": 2.5,
                   "c4dsfft": 45.0, "c5": 0.5}


def import_reference():
    """The installed reference package, or None when baseline/_ref is absent."""
    if not os.path.isdir(os.path.join(REF_DIR, "aliasfft")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    sys.dont_write_bytecode = True
    import aliasfft

    # the reference's 64x64 small-matrix cap makes R-FFAST / noisy DSFFT
    # raise above N = 2^21; lifted at runtime (its files untouched)
    sys.modules["aliasfft.smallnum"].MAX_DIM = 4096
    return aliasfft


def reference_call(ref, name, x, seed):
    """One signal through the reference's public API."""
    cfg = REF_CONFIGS[name]
    n, k = cfg["n"], cfg["k"]
    if name in ("c1", "c5"):
        from aliasfft.oneshot import truncate_spectrum
        from aliasfft.peeling import build_graph, exact_thresholds, peel_decode

        factors = [49, 50, 51] if name == "c1" else FACTORS
        g = build_graph(x, ref.CyclePlan(factors, [0, 1, 2]))
        e = exact_thresholds(x)
        r = peel_decode(g, "exact", eps_zero=e, eps_ratio=e, max_rounds=k + 4)
        return truncate_spectrum(r.spectrum.entries, n, k)
    if name in ("c2", "c4dt3"):
        b, variant = (1024, "dt2") if name == "c2" else (4096, "dt3")
        return ref.sfft_dt(x, k, ref.OneShotConfig(b=b, a_m=4, p=15, variant=variant, seed=seed))
    if name in ("c3", "c3auto"):
        from aliasfft.oneshot import truncate_spectrum
        from aliasfft.peeling import build_graph, noisy_thresholds, peel_decode

        plan, sp = ref.plan_cycles(n, k, "noisy", seed)
        factors = [511, 512, 513] if name == "c3" else list(plan.factors)
        g = build_graph(x, ref.CyclePlan(factors, sp.shifts))
        sp.t0, sp.t1 = noisy_thresholds(g)
        r = peel_decode(g, "noisy", search_plan=sp, max_rounds=k + 4)
        return truncate_spectrum(r.spectrum.entries, n, k)
    if name == "c4dsfft":
        snr = cfg["snr"]
        return ref.dsfft(x, k, ref.DsfftConfig(mode="noisy", seed=seed,
                                               noise_std=float(np.sqrt(k * 10 ** (-snr / 10)))))
    raise ValueError(name)


def _ref_cpu_worker(name, trials, barrier, q, use_port=False):
    """Generate this worker's signals (not timed, bench.py:172-176), then time each
    reference call; reports [(start, end), ...] in perf_counter seconds."""
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"
    try:
        cfg = REF_CONFIGS[name]
        n, k, snr = cfg["n"], cfg["k"], cfg["snr"]
        ref = None if use_port else import_reference()
        if ref is not None:
            gen = ref.generate_test_case
        else:
            from paper_2011_05749_b200.signals import generate_test_case as gen
        xs = []
        for t in trials:
            seed = case_seed(n, k, snr, 0, t)
            x = gen(n, k, snr, seed).signal
            if cfg["c64"]:  # the reference upcasts c64 input to c128 (bucketize.py:91)
                x = x.astype(np.complex64).astype(np.complex128)
            xs.append((seed, x))
        if ref is None:
            from oracle import ffast as oracle_ffast

            def call(x, seed):
                return oracle_ffast.ffast(x, k, [49, 50, 51] if name == "c1" else FACTORS)
        else:
            def call(x, seed):
                return reference_call(ref, name, x, seed)
        if barrier is not None:
            barrier.wait()
        out = []
        for seed, x in xs:
            t0 = time.perf_counter()
            call(x, seed)
            out.append((t0, time.perf_counter()))
        q.put(("ok", out))
    except Exception as exc:  # pragma: no cover - reported, not raised
        q.put(("error", f"{type(exc).__name__}: {exc}"))


def _run_pool(name, per_worker, workers, first_trial=0, use_port=False):
    import multiprocessing as mp

    # the spawned children import numpy (at bench.py's top) before the worker body
    # runs: their BLAS / OpenMP thread counts must already be in the environment
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    barrier = ctx.Barrier(workers) if workers > 1 else None
    procs = []
    for w in range(workers):
        trials = [first_trial + w * per_worker + j for j in range(per_worker)]
        p = ctx.Process(target=_ref_cpu_worker, args=(name, trials, barrier, q, use_port))
        p.start()
        procs.append(p)
    res = [q.get() for _ in procs]
    for p in procs:
        p.join()
    errs = [r[1] for r in res if r[0] != "ok"]
    if errs:
        raise RuntimeError(errs[0])
    return [r[1] for r in res]


def ref_cpu_baseline(name, one_core_signals, per_core_signals, max_workers=None,
                     use_port=False):
    """The reference timed on this host: (i) a 1-core median per signal (one process
    alone, OMP/OpenBLAS threads = 1), (ii) all-core throughput (one process per core,
    each timing its own signals, started together; total signals over the union of
    their timed spans).  Signal generation is excluded (bench.py:172-176)."""
    cores = os.cpu_count() or 1
    workers = cores
    try:
        import psutil

        avail = psutil.virtual_memory().available / 2**30
        workers = max(1, min(workers, int(0.8 * avail / REF_GB_PER_PROC[name])))
    except Exception:
        pass
    if max_workers:
        workers = min(workers, max_workers)
    t_start = time.perf_counter()
    one = _run_pool(name, one_core_signals, 1, first_trial=0, use_port=use_port)[0]
    durs = [b - a for a, b in one]
    allc = _run_pool(name, per_core_signals, workers, first_trial=one_core_signals,
                     use_port=use_port)
    t0 = min(s[0][0] for s in allc)
    t1 = max(s[-1][1] for s in allc)
    total = workers * per_core_signals
    kind = "port" if use_port or import_reference() is None else "reference"
    return {
        "value": total / (t1 - t0), "unit": UNIT, "cores": workers, "kind": kind,
        "one_core_median_s": statistics.median(durs),
        "one_core_signals_per_s": 1.0 / statistics.median(durs),
        "sample": (f"{name}: 1-core median over {one_core_signals} signal(s); all-core "
                   f"throughput {workers} processes x {per_core_signals} signal(s) "
                   f"(trials {one_core_signals}..{one_core_signals + total - 1}); "
                   + ("reference package baseline/_ref, SURVEY Appendix A call"
                      if kind == "reference" else "oracle numpy port")
                   + "; OMP/OpenBLAS threads 1; generation excluded"),
        "wall_s": time.perf_counter() - t_start,
    }


# ============================================================================ device inputs


def synth_batch(n, k, snr, trials, dtype, dev, chunk=8):
    """Signals for the given trials: numpy-PCG64 truth (the reference's draw order),
    n * ifft on the device, Gaussian noise at `snr` drawn on the device."""
    import torch

    from paper_2011_05749_b200.signals import draw_truth

    x = torch.empty((len(trials), n), dtype=dtype, device=dev)
    truths = []
    for c0 in range(0, len(trials), chunk):
        c1 = min(len(trials), c0 + chunk)
        spec = torch.zeros((c1 - c0, n), dtype=torch.complex128, device=dev)
        for i in range(c0, c1):
            rng = np.random.default_rng(case_seed(n, k, snr, 0, trials[i]))
            pos, coef = draw_truth(n, k, rng)
            truths.append(pos)
            spec[i - c0, torch.from_numpy(pos).to(dev)] = torch.from_numpy(coef).to(dev)
        sig = torch.fft.ifft(spec, dim=1)
        del spec
        sig *= n
        if snr != "exact":
            p_sig = (sig.abs() ** 2).mean(dim=1, keepdim=True)
            std = torch.sqrt(p_sig / 10 ** (float(snr) / 10) / 2)
            g = torch.Generator(device=dev).manual_seed(1000003 * trials[c0] + 17)
            noise = torch.randn((c1 - c0, n, 2), device=dev, generator=g, dtype=torch.float64)
            sig += std * torch.view_as_complex(noise)
            del noise
        x[c0:c1] = sig.to(dtype)
        del sig
    torch.cuda.synchronize()
    return x, truths


def synth_signals(x, first_trial: int, dev, chunk: int = 32):
    """Fill a preallocated [count, N] config-5 batch with trials first_trial.. (tools/)."""
    truths = []
    for c0 in range(0, x.shape[0], chunk):
        c1 = min(x.shape[0], c0 + chunk)
        xs, tr = synth_batch(N_SIG, K, "exact", list(range(first_trial + c0, first_trial + c1)),
                             x.dtype, dev, chunk=chunk)
        x[c0:c1] = xs
        truths += tr
        del xs
    return truths


# ============================================================================ our arm


def run_ours(args, world, rank, local):
    import torch
    import torch.distributed as dist

    from paper_2011_05749_b200 import _lib
    from paper_2011_05749_b200.batch import ffast_batch, ffast_workspace_bytes

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        # NCCL's communicator INIT lines (nranks per comm) on stderr, also when the
        # driver launches torchrun itself
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        dist.init_process_group("nccl", device_id=dev)
    from paper_2011_05749_b200.shard import gather_slots, max_over_ranks, shard_range

    total = args.signals
    if total % world:
        raise SystemExit("--total-signals must be a multiple of the rank count (equal result slots)")
    first, stop = shard_range(total, rank, world)
    per = stop - first

    x, truths = synth_batch(N_SIG, K, "exact", list(range(first, stop)), torch.complex64, dev,
                            chunk=32)
    lib = _lib.load()  # noqa: F841  (fail loudly here if the library is missing)
    code = _lib.AFFT_C64
    ws = torch.empty(ffast_workspace_bytes(N_SIG, code, per, FACTORS), dtype=torch.uint8,
                     device=dev)
    res = ffast_batch(x, K, FACTORS, workspace=ws)
    stream = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    gathered = {}

    def step(i=None):
        """One FFAST pass over the resident batch: a single afft_ffast call (one
        ffast_fused_kernel or ffast_parts_kernel launch), then the NCCL gather of the
        result slots."""
        if i is not None:
            ev[i][0].record(stream)
        ffast_batch(x, K, FACTORS, workspace=ws, out=res)
        if i is not None:
            ev[i][1].record(stream)
        if world > 1:
            gathered["slots"] = gather_slots(res.pos, res.val, res.count)

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
    exact = sum(int(cnt[i]) == K and set(pos[i, :K].tolist()) == set(truths[i].tolist())
                for i in range(per))
    kept = sum(int(c) for c in cnt)
    true_kept = sum(len(set(pos[i, :int(cnt[i])].tolist()) & set(truths[i].tolist()))
                    for i in range(per))
    if world > 1:
        # the gathered slots carry every rank's results in rank order
        gp, _, gc = gathered["slots"]
        assert gp.shape[0] == total and int(gc.sum()) > 0
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
    stats = max_over_ranks([per - exact, kept - true_kept], dev)

    # e2e on every rank at once (each GPU has its own PCIe link): whole-job signals over
    # the slowest rank's time
    if world > 1:
        dist.barrier()
    e2e = run_e2e(args, dev, x)
    e2e_ms, copy_ms = max_over_ranks([e2e["ms_per_step"], e2e.pop("_copy_ms")], dev)
    e2e.update({"value": world * e2e["signals_per_step"] / (e2e_ms * 1e-3),
                "ms_per_step": e2e_ms, "signals_per_step": world * e2e["signals_per_step"],
                "h2d_bytes_per_step": world * e2e["h2d_bytes_per_step"],
                "d2h_bytes_per_step": world * e2e["d2h_bytes_per_step"],
                "frac_of_h2d_bound": copy_ms / e2e_ms, "ranks": world})
    read_gbs = read_stream_gbs(x, dev) if rank == 0 else None
    context = dense_fft_context(x, dev) if (rank == 0 and not args.quick) else None
    del x, ws
    torch.cuda.empty_cache()
    if world > 1:
        dist.barrier()

    cpu = None
    configs = None
    if rank == 0:
        if not args.quick:
            cpu = ref_cpu_baseline("c5", 5, 4)
            port = ref_cpu_baseline("c5", 5, 4, use_port=True)
            cpu["port"] = {"value": port["value"], "cores": port["cores"],
                           "one_core_signals_per_s": port["one_core_signals_per_s"],
                           "sample": port["sample"]}
            cpu["host"] = host_info()
        if world == 1 and not args.no_configs:
            configs = run_configs(dev, args)
    if world > 1:
        dist.barrier()

    if rank == 0:
        peak, peak_src = load_peaks()
        gsec = gather_sector_bytes()
        alg_bytes = per * (SIGNAL_BYTES + gsec)
        achieved = alg_bytes / (kern_ms * 1e-3) / 1e9
        traffic = None
        d = load_json("ncu_ffast_fused_traffic.json")
        if d:
            traffic = float(d["dram_bytes_per_signal"]) * per
        value = total / (ms_per_step * 1e-3)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "c64 in, f64 compute", "data": "synthetic (generate_test_case model, seeded)",
            "config": config_dict(world, total),
            "roofline": {
                "kernel": f"{kernel_name} (|x|^2 stream + gather/DFT + peel + truncate)",
                "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "peak_source": peak_src,
                "algorithmic_bytes_per_launch": alg_bytes, "traffic": traffic,
                "algorithmic_bytes_per_signal": SIGNAL_BYTES + gsec,
                "gather_sector_bytes_per_signal": gsec,
                "launch_ms": kern_ms,
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
            "checks": {"signals_not_exact_max_rank": stats[0],
                       "false_tones_max_rank": stats[1],
                       "exact_recovered_fraction_rank0": exact / per,
                       "true_tone_fraction_rank0": true_kept / max(1, kept),
                       "step": ("one ffast_fused_kernel launch per step (afft_ffast mode 0)"
                                if fused else
                                "one ffast_parts_kernel launch per step (afft_ffast mode 4: "
                                "several CTAs stream parts of each signal's |x|^2, the last "
                                "one decodes it)")},
            "nccl": ({"backend": "nccl", "comm_nranks": world,
                      "collective": "all_gather_into_tensor of the [signals, K] result slots"}
                     if world > 1 else None),
            "context": context,
            "configs": configs,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def config_dict(world, total=TOTAL_SIGNALS):
    """The headline workload, identical in both arms."""
    return {
        "workload": WORKLOAD, "n": N_SIG, "k": K, "factors": FACTORS, "shifts": [0, 1, 2],
        "signals_total": total, "signals_per_rank": total // world,
        "l2": "inputs 137 GB >> 126 MB L2 (no flush needed)",
        "parallelism": f"signal-sharded x{world}, NCCL all-gather of result slots",
    }


def dist_ready() -> bool:
    import torch.distributed as dist

    return dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1


def run_e2e(args, dev, x):
    """Same metric through the public API with HOST (pinned) buffers: H2D of every
    step's signals + the decode + D2H of the result slots, all timed.  Per rank; the
    caller combines the ranks (max time)."""
    import torch

    from paper_2011_05749_b200.batch import ffast_batch

    m = min(args.e2e_signals, x.shape[0])
    while True:  # pinned host staging; a host that cannot lock this much gets half
        try:
            host = torch.empty((m, N_SIG), dtype=torch.complex64, pin_memory=True)
            break
        except (RuntimeError, torch.AcceleratorError) if hasattr(torch, "AcceleratorError") \
                else RuntimeError:
            if m <= 16:
                raise
            m //= 2
            print(f"bench: pinned staging failed, e2e with {m} signals per step",
                  file=sys.stderr)
    if dist_ready():  # every rank stages the same count (the line reports world x m)
        mt = torch.tensor([m], dtype=torch.int64, device=dev)
        torch.distributed.all_reduce(mt, op=torch.distributed.ReduceOp.MIN)
        m = int(mt.item())
        host = host[:m]  # a view of the pinned block
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
    del dbuf, host
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
    B200 (via torch, c64 and c128), this library's K2' (b = N) and numpy on one host
    core — in signals/s."""
    import torch

    from paper_2011_05749_b200 import _device, _lib

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

    m = min(512, x.shape[0])
    xs = x[:m]
    out = torch.empty_like(xs)
    gpu_ms = timed(lambda: out.copy_(torch.fft.fft(xs, dim=1)))
    del out
    m2 = min(64, x.shape[0])
    x2 = x[:m2]
    x2c = x2.to(torch.complex128)
    out2 = torch.empty((m2, N_SIG), dtype=torch.complex128, device=dev)
    lib = _lib.load()
    sb, ns = _lib.host_i64([0])

    def run_c128():
        out2.copy_(torch.fft.fft(x2c, dim=1))

    def run_k2():
        _lib.check(lib.afft_bucketize(x2.data_ptr(), _device.dtype_code(x2), N_SIG, m2, N_SIG,
                                      N_SIG, sb, ns, out2.data_ptr(), N_SIG, N_SIG, 1,
                                      _device.stream_ptr()), "bucketize(b=N)")

    c128_ms = timed(run_c128)
    ours_ms = timed(run_k2)
    del x2c, out2
    host = x[0].cpu().numpy()
    t0 = time.perf_counter()
    for _ in range(3):
        np.fft.fft(host.astype(np.complex128))
    cpu_s = (time.perf_counter() - t0) / 3
    return {"dense_fft_gpu_signals_per_s": m / (gpu_ms * 1e-3), "dense_fft_gpu": "cuFFT c64 (torch.fft)",
            "dense_fft_gpu_c128_signals_per_s": m2 / (c128_ms * 1e-3),
            "dense_fft_ours_signals_per_s": m2 / (ours_ms * 1e-3),
            "dense_fft_ours": "K2' (afft_bucketize, b = N), c64 in, f64 compute, c128 out",
            "dense_fft_cpu_signals_per_s": 1.0 / cpu_s, "dense_fft_cpu": "numpy pocketfft c128, 1 core",
            "note": "context only; not part of the measured path"}


# ============================================================================ configs 1-4


def _timed(fn, reps):
    """Mean ms per call over `reps` calls after one warm-up, CUDA events on the
    caller's stream (the batched entry points join any helper streams back to it)."""
    import torch

    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def _recall(found_sets, truths):
    hits = sum(len(set(f) & set(t.tolist())) for f, t in zip(found_sets, truths))
    return hits / max(1, sum(len(t) for t in truths))


def _fp64_roofline(name, signals, ms, pipes, fp64_peak, fp64_src):
    """FP64 roofline of a compute-bound config from its ncu-counted FP64 work per
    signal (profiles/r02_pipes.json: sass dadd + dmul + 2 dfma over every kernel of one
    batched call) over the live CUDA-event time."""
    entry = (pipes or {}).get(name)
    if not entry:
        return {"bound": "fp64", "achieved": None, "peak": fp64_peak, "unit": "TFLOP/s",
                "frac": None, "note": "profiles/r02_pipes.json has no entry for this config"}
    flops = float(entry["fp64_flops_per_signal"]) * signals
    ach = flops / (ms * 1e-3) / 1e12
    return {"bound": "fp64", "achieved": ach, "peak": fp64_peak, "unit": "TFLOP/s",
            "frac": ach / fp64_peak, "peak_source": fp64_src,
            "fp64_flops_per_signal": entry["fp64_flops_per_signal"],
            "dominant_kernel": entry.get("dominant_kernel"),
            "dominant_fp64_pipe_pct": entry.get("dominant_fp64_pipe_pct"),
            "dominant_issue_pct": entry.get("dominant_issue_pct"),
            "source": "ncu counts (tools/ncu_pipes.py -> profiles/r02_pipes.json) over live time"}


def run_configs(dev, args):
    """Configs 1-4 on this GPU, each with its roofline and the reference's CPU time."""
    import torch

    from paper_2011_05749_b200 import (
        DsfftConfig, ffast_batch, plan_cycles, rffast_batch, sfft_dt_batch,
    )
    from paper_2011_05749_b200.dsfft import dsfft_batch

    peak, peak_src = load_peaks()
    fp64_peak, fp64_src = load_fp64_peak()
    pipes = load_json("r02_pipes.json")
    committed_cpu = load_json("r02_ref_cpu.json") or {}
    reps = max(2, min(args.steps, 5))
    out = {}

    def cpu_for(name, one, per):
        if args.quick:
            return None
        if name in committed_cpu:
            d = dict(committed_cpu[name])
            d["source"] = ("committed measurement on a B200 box's host "
                           "(python bench.py --ref-cpu ..., profiles/r02_ref_cpu.json); too "
                           "slow to re-run inside every bench")
            return d
        if name in ("c3", "c3auto", "c4dsfft"):
            return None
        return ref_cpu_baseline(name, one, per)

    # ---- C1: FFAST exact, N = 49*50*51, K = 40, c128 (one signal is us-scale: a batch
    # of seeded signals measures throughput; the single-signal latency is a CUDA graph)
    n, k, f = 124950, 40, [49, 50, 51]
    S = 8192
    x, tr = synth_batch(n, k, "exact", list(range(S)), torch.complex128, dev, chunk=512)
    ws = torch.empty(1 << 24, dtype=torch.uint8, device=dev)
    res = ffast_batch(x, k, f, workspace=ws)
    ms = _timed(lambda: ffast_batch(x, k, f, workspace=ws, out=res), reps)
    one = x[:1].clone()
    r1 = ffast_batch(one, k, f)
    ffast_batch(one, k, f, workspace=ws, out=r1)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ffast_batch(one, k, f, workspace=ws, out=r1)
    one_ms = _timed(g.replay, 50)
    bytes_sig = n * 16 + gather_sector_bytes(n, f, esz=16)
    ach = S * bytes_sig / (ms * 1e-3) / 1e9
    cnt = res.count.cpu().numpy()
    posn = res.pos.cpu().numpy()
    out["c1"] = {
        "workload": "config1_ffast_n124950_k40_49x50x51_c128", "signals": S,
        "value": S / (ms * 1e-3), "unit": UNIT, "ms": ms, "single_signal_us": one_ms * 1e3,
        "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                     "frac": ach / peak, "peak_source": peak_src,
                     "algorithmic_bytes_per_signal": bytes_sig,
                     "note": "|x|^2 pass (2.0 MB c128) + gather sectors"},
        "check": {"recall": _recall([posn[i, :cnt[i]] for i in range(S)], tr)},
        "cpu_baseline": cpu_for("c1", 20, 20),
    }
    del x, res, ws, one, r1, g
    torch.cuda.empty_cache()

    # ---- C2: sFFT-DT2, N = 2^22, K = 1000, B = 1024, p = 15, 64 signals, c128
    n, k, S = 1 << 22, 1000, 64
    x, tr = synth_batch(n, k, "exact", list(range(S)), torch.complex128, dev, chunk=16)
    seeds = [case_seed(n, k, "exact", 0, i) for i in range(S)]
    res = sfft_dt_batch(x, k, 1024, 4, 15, "dt2", seeds=seeds)
    ms = _timed(lambda: sfft_dt_batch(x, k, 1024, 4, 15, "dt2", seeds=seeds), reps)
    cnt = res.count.cpu().numpy()
    posn = res.pos.cpu().numpy()
    sec = gather_sector_bytes(n, [1024], shifts=list(range(-4, 8)), esz=16)
    out["c2"] = {
        "workload": "config2_sfftdt2_n4194304_k1000_b1024_p15_c128", "signals": S,
        "value": S / (ms * 1e-3), "unit": UNIT, "ms": ms,
        "roofline": _fp64_roofline("c2", S, ms, pipes, fp64_peak, fp64_src),
        "hbm_view": {"structured_sector_bytes_per_signal": sec,
                     "achieved_gbs": S * sec / (ms * 1e-3) / 1e9,
                     "note": "sector bytes of the 12 structured shifts only (random shifts "
                             "add 15 more cosets); far below HBM: not the bound"},
        "check": {"recall": _recall([posn[i, :cnt[i]] for i in range(S)], tr)},
        "cpu_baseline": cpu_for("c2", 3, 1),
    }
    del x, res
    torch.cuda.empty_cache()

    # ---- C3: R-FFAST, N = 511*512*513, K = 1000, 20 dB, 16 signals, c128; the literal
    # 511/512/513 plan and the reference's auto plan, per-signal search plans
    n, k, S = 511 * 512 * 513, 1000, 16
    x, tr = synth_batch(n, k, 20.0, list(range(S)), torch.complex128, dev, chunk=2)
    seeds = [case_seed(n, k, 20.0, 0, i) for i in range(S)]
    plans = [plan_cycles(n, k, "noisy", seed=s) for s in seeds]
    for name, factors in (("c3", [511, 512, 513]), ("c3auto", list(plans[0][0].factors))):
        searches = [p[1] for p in plans]  # each signal's own anchors (peeling.py:163-164)
        res = rffast_batch(x, k, factors, searches)
        ms = _timed(lambda: rffast_batch(x, k, factors, searches), reps)
        cnt = res.count.cpu().numpy()
        posn = res.pos.cpu().numpy()
        out[name] = {
            "workload": f"config3_rffast_n134217216_k1000_20db_{'x'.join(map(str, factors))}_c128",
            "signals": S, "value": S / (ms * 1e-3), "unit": UNIT, "ms": ms,
            "roofline": _fp64_roofline(name, S, ms, pipes, fp64_peak, fp64_src),
            "check": {"recall": _recall([posn[i, :cnt[i]] for i in range(S)], tr),
                      "rounds": sorted(set(int(r) for r in res.rounds.cpu().tolist()))},
            "cpu_baseline": cpu_for(name, 1, 1),
        }
    del x, res
    torch.cuda.empty_cache()

    # ---- C4: N = 2^24, K = 4096, c64, SNR 10/20/30 dB, 32 signals per SNR:
    # sFFT-DT3 (B = 4096, p = 15) and DSFFT (noise_std = sqrt(K 10^(-snr/10)))
    n, k, S = 1 << 24, 4096, 32
    dt_ms, ds_ms, dt_rec, ds_rec, ds_nat_ms, ds_nat_fb, ds_nat4_ms = {}, {}, {}, {}, {}, {}, {}
    from paper_2011_05749_b200.dsfft import _dsfft_batch_native, _on_worker_streams
    for snr in (10.0, 20.0, 30.0):
        x, tr = synth_batch(n, k, snr, list(range(S)), torch.complex64, dev, chunk=4)
        seeds = [case_seed(n, k, snr, 0, i) for i in range(S)]
        res = sfft_dt_batch(x, k, 4096, 4, 15, "dt3", seeds=seeds)
        dt_ms[snr] = _timed(lambda: sfft_dt_batch(x, k, 4096, 4, 15, "dt3", seeds=seeds), reps)
        cnt = res.count.cpu().numpy()
        posn = res.pos.cpu().numpy()
        dt_rec[snr] = _recall([posn[i, :cnt[i]] for i in range(S)], tr)
        cfgs = [DsfftConfig(mode="noisy", seed=s, noise_std=float(np.sqrt(k * 10 ** (-snr / 10))))
                for s in seeds]
        outs = dsfft_batch(x, k, cfgs)
        ds_ms[snr] = _timed(lambda: dsfft_batch(x, k, cfgs), reps)
        ds_rec[snr] = _recall([np.array(list(o.entries)) for o in outs], tr)
        # the C ABI in lockstep (afft_dsfft_batch: entries as arrays, no Python dicts)
        nat = _dsfft_batch_native(x, k, cfgs, list(range(S)))
        ds_nat_fb[snr] = S - len(nat)
        ds_nat_ms[snr] = _timed(lambda: _dsfft_batch_native(x, k, cfgs, list(range(S))),
                                reps)
        # the same C ABI call on 8 worker streams x 4 signals (one group's read-backs and
        # small kernels overlap another's spectrum passes; tools/dsfft_lockstep_sweep.py)
        parts = [list(range(c0, min(S, c0 + 4))) for c0 in range(0, S, 4)]
        ds_nat4_ms[snr] = _timed(
            lambda: _on_worker_streams(x, parts, 8,
                                       lambda part: _dsfft_batch_native(x, k, cfgs, part)),
            reps)
        del x, res
        torch.cuda.empty_cache()
    tot_dt = sum(dt_ms.values())
    out["c4dt3"] = {
        "workload": "config4_sfftdt3_n16777216_k4096_b4096_p15_c64_10-20-30db",
        "signals": 3 * S, "value": 3 * S / (tot_dt * 1e-3), "unit": UNIT,
        "ms_per_snr": {f"{int(s)}db": v for s, v in dt_ms.items()},
        "roofline": _fp64_roofline("c4dt3", 3 * S, tot_dt, pipes, fp64_peak, fp64_src),
        "check": {"recall_per_snr": {f"{int(s)}db": v for s, v in dt_rec.items()},
                  "note": "degenerate on the reference too (SURVEY Appendix A: l0 7347-8032)"},
        "cpu_baseline": cpu_for("c4dt3", 2, 1),
    }
    tot_ds = sum(ds_ms.values())
    floor = n * (8 + 16) + 2 * n * 32
    ach = 3 * S * floor / (tot_ds * 1e-3) / 1e9
    out["c4dsfft"] = {
        "workload": "config4_dsfft_n16777216_k4096_c64_10-20-30db",
        "signals": 3 * S, "value": 3 * S / (tot_ds * 1e-3), "unit": UNIT,
        "ms_per_snr": {f"{int(s)}db": v for s, v in ds_ms.items()},
        "api": "dsfft_batch (lockstep chunks of <= 4 signals on 8 worker streams, guided sizes; SparseSpectrum dicts built on the calling thread)",
        "native_lockstep": {
            "value": 3 * S / (sum(ds_nat_ms.values()) * 1e-3), "unit": UNIT,
            "ms_per_snr": {f"{int(s)}db": v for s, v in ds_nat_ms.items()},
            "fallback_signals": {f"{int(s)}db": v for s, v in ds_nat_fb.items()},
            "streams_8x4": {"value": 3 * S / (sum(ds_nat4_ms.values()) * 1e-3), "unit": UNIT,
                            "ms_per_snr": {f"{int(s)}db": v for s, v in ds_nat4_ms.items()},
                            "api": "afft_dsfft_batch, 4 signals per call on 8 worker streams"},
            "api": "afft_dsfft_batch (C ABI, lockstep, entries as arrays before truncation)"},
        "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                     "frac": ach / peak, "peak_source": peak_src,
                     "algorithmic_bytes_per_signal": floor,
                     "c_abi_streams_8x4_frac": 3 * S * floor / (sum(ds_nat4_ms.values()) * 1e-3)
                     / 1e9 / peak,
                     "note": "floor traffic: a three-pass 2^24 FFT to the resident c128 "
                             "spectrum (first pass reads c64; the |x|^2 norm and the deep "
                             "layers' active sets ride on its last pass)"},
        "check": {"recall_per_snr": {f"{int(s)}db": v for s, v in ds_rec.items()}},
        "cpu_baseline": cpu_for("c4dsfft", 1, 1),
    }
    return out


# ============================================================================ reference arm


def run_reference(args, world, rank):
    """The reference package itself (baseline/_ref) on all host cores, headline workload.
    Under torchrun only rank 0 works; the others exit without work."""
    if rank != 0:
        return
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"
    use_port = import_reference() is None
    cores = os.cpu_count() or 1
    per_step = 4  # signals per core per step: amortises the per-step barrier
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    barrier = ctx.Barrier(cores)
    steps = args.steps + args.warmup
    procs = [ctx.Process(target=_ref_step_worker,
                         args=(w, per_step, steps, barrier, q, use_port))
             for w in range(cores)]
    for p in procs:
        p.start()
    results = [q.get() for _ in procs]
    for p in procs:
        p.join()
    errs = [r for r in results if isinstance(r, str)]
    if errs:
        raise SystemExit(errs[0])
    step_ms = []
    for s in range(args.warmup, steps):
        t0 = min(r[s][0] for r in results)
        t1 = max(r[s][1] for r in results)
        step_ms.append((t1 - t0) * 1e3)
    ms = statistics.mean(step_ms)
    value = cores * per_step / (ms * 1e-3)
    kind = "port" if use_port else "reference"
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "c64 in, f64 compute (the reference upcasts to c128)",
        "data": "synthetic (generate_test_case model, seeded)", "impl": "reference",
        "config": config_dict(world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": f"{cores * per_step} signals per step ({per_step} per core, "
                                   "one process per core), "
                                   + ("the reference package (baseline/_ref) through its "
                                      "public API, SURVEY Appendix A config-5 call"
                                      if kind == "reference" else
                                      "oracle/ffast.py (baseline/_ref missing)")
                                   + "; signal generation excluded as bench.py:172-176 does",
                         "host": host_info()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _ref_step_worker(wid, per_step, steps, barrier, q, use_port):
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"
    try:
        ref = None if use_port else import_reference()
        if ref is not None:
            gen = ref.generate_test_case
        else:
            from paper_2011_05749_b200.signals import generate_test_case as gen
            from oracle import ffast as oracle_ffast
        xs = []
        for j in range(per_step):
            seed = case_seed(N_SIG, K, "exact", 0, wid * per_step + j)
            xs.append((seed, gen(N_SIG, K, "exact", seed).signal.astype(np.complex64)
                       .astype(np.complex128)))
        times = []
        for _ in range(steps):
            barrier.wait()
            t0 = time.perf_counter()
            for seed, x in xs:
                if ref is not None:
                    reference_call(ref, "c5", x, seed)
                else:
                    oracle_ffast.ffast(x, K, FACTORS)
            times.append((t0, time.perf_counter()))
        q.put(times)
    except Exception as exc:  # pragma: no cover
        q.put(f"{type(exc).__name__}: {exc}")


# ============================================================================ dry run


def run_dry(args, world, rank):
    """The multi-rank plumbing without a GPU (tests/test_bench_launcher.py): gloo
    process group, the same signal sharding, result-slot all-gather and max-over-ranks
    timing as run_ours, over stand-in result slots (slot values derived from the global
    signal index, so the gathered order is checkable).  No decode runs; the line says
    so with "dry_run": true."""
    import torch
    import torch.distributed as dist

    from paper_2011_05749_b200.shard import gather_slots, max_over_ranks, shard_range

    if world > 1:
        dist.init_process_group("gloo")
    total = args.signals
    if total % world:
        raise SystemExit("--total-signals must be a multiple of the rank count (equal result slots)")
    first, stop = shard_range(total, rank, world)
    per = stop - first
    idx = torch.arange(first, stop, dtype=torch.int64)
    pos = idx[:, None] * 1000 + torch.arange(K, dtype=torch.int64)[None, :]
    val = torch.complex(idx[:, None].double().expand(per, K), torch.zeros(per, K, dtype=torch.float64))
    cnt = torch.full((per,), K, dtype=torch.int32)
    t0 = time.perf_counter()
    gp, gv, gc = gather_slots(pos, val, cnt) if world > 1 else (pos, val, cnt)
    ms = (time.perf_counter() - t0) * 1e3
    ok = (gp.shape[0] == total and bool((gp[:, 0] == torch.arange(total) * 1000).all())
          and bool((gv[:, 0].real == torch.arange(total).double()).all())
          and int(gc.sum()) == total * K)
    (ms_max,) = max_over_ranks([ms], torch.device("cpu"))
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": None, "unit": UNIT, "n_gpus": world, "dry_run": True,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
            "higher_is_better": True, "scaling": "strong", "config": config_dict(world, total),
            "checks": {"gathered_slots_in_rank_order": ok, "signals_per_rank": per},
        }), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ============================================================================ entry


def relaunch_under_torchrun(args_list, n):
    """--gpus N > 1 without a torchrun environment: one rank per GPU via
    torch.distributed.run on 127.0.0.1; rank 0's JSON line is passed through."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + args_list
    return subprocess.run(cmd, env=env).returncode


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--total-signals", dest="signals", type=int, default=TOTAL_SIGNALS)
    ap.add_argument("--e2e-signals", type=int, default=256)
    ap.add_argument("--no-configs", action="store_true", help="skip configs 1-4 at N=1")
    ap.add_argument("--quick", action="store_true",
                    help="skip the CPU baselines and the dense-FFT context")
    ap.add_argument("--ref-cpu", default=None,
                    help="only time the reference on this host for these configs "
                         "(comma list) and write --ref-cpu-out")
    ap.add_argument("--ref-cpu-out", default=os.path.join(ROOT, "profiles", "r02_ref_cpu.json"))
    ap.add_argument("--dry-run", action="store_true",
                    help="exercise the launcher / sharding / gather plumbing on CPU (gloo)")
    argv = sys.argv[1:] if argv is None else argv
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3
    if args.ref_cpu:
        plan = {"c3": (1, 1), "c3auto": (1, 1), "c4dsfft": (1, 1), "c4dt3": (2, 1),
                "c2": (3, 1), "c1": (20, 20), "c5": (5, 4)}
        out = load_json(os.path.basename(args.ref_cpu_out)) or {}
        for name in args.ref_cpu.split(","):
            one, per = plan[name]
            out[name] = ref_cpu_baseline(name, one, per)
            out[name]["host"] = host_info()
            with open(args.ref_cpu_out, "w") as fh:
                json.dump(out, fh, indent=1)
            print(json.dumps({name: out[name]}), flush=True)
        return 0
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None and args.gpus > 1:
        return relaunch_under_torchrun(argv, args.gpus)
    world = int(env_world or "1")
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    if args.dry_run:
        run_dry(args, world, rank)
    elif args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)
    return 0


if __name__ == "__main__":
    sys.exit(main())
