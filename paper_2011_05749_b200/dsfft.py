"""Deterministic binary-tree search (DSFFT) on the GPU.

Drop-in for /root/reference/pkg/src/aliasfft/dsfft.py.  `dsfft` runs the whole
layer loop natively (afft_dsfft, csrc/dsfft_host.cu: one read-back per layer);
every layer's data stays on the device: full layers are size-2^d bucketizations,
selective layers are direct alias sums, deep layers read the resident spectrum
through the alias identity, activity is a device stream compaction,
classification reuses the exact / noisy singleton kernels on measurement rows
built with coset reuse (csrc/dsfft.cu), and leftover aliased buckets go through
the sFFT-DT3 kernels.  This module draws the numpy-PCG64 inputs, replays the
ledger, and keeps the reference's layer-level API (initial_layer / expand_layer).
"""

from __future__ import annotations

import ctypes
import os
import functools
import warnings
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device, _lib
from .bucketize import SampleLedger, gather_indices, record_bucketization
from .oneshot import OneShotConfig, random_shifts, structured_shifts
from .peeling import SearchPlan, UnsupportedSizeError, kay_weights
from .signals import SparseSpectrum



@dataclass
class TreeLayer:
    """One layer: computed bucket values and the active set (dsfft.py:42-56)."""

    depth: int
    values: dict[int, complex]
    active: set[int] = field(default_factory=set)

    @property
    def b(self) -> int:
        return 1 << self.depth

    @property
    def m_d(self) -> int:
        return len(self.active)


@dataclass
class DsfftConfig:
    theta: float = 0.75
    mode: str = "exact"
    a_m: int = 4
    seed: int = 0
    noise_std: float = 0.0
    activity_floor: float = 1e-6


# ------------------------------------------------------------------ device layer


@dataclass
class _DevLayer:
    depth: int
    active: torch.Tensor  # ascending bucket indices (device int64)
    values: torch.Tensor | None = None  # full layer: [b] complex128; selective: [ncand]
    cand: torch.Tensor | None = None    # selective layer: candidate bucket indices

    @property
    def b(self) -> int:
        return 1 << self.depth

    @property
    def m_d(self) -> int:
        return int(self.active.numel())


def _active(values: torch.Tensor, thr: float, cand: torch.Tensor | None = None) -> torch.Tensor:
    count = torch.zeros(1, dtype=torch.int32, device=values.device)
    out = torch.empty(values.numel(), dtype=torch.int64, device=values.device)
    _lib.check(
        _lib.load().afft_active_indices(values.data_ptr(), values.numel(), float(thr),
                                        None if cand is None else cand.data_ptr(),
                                        out.data_ptr(), count.data_ptr(), _device.stream_ptr()),
        "active_indices",
    )
    return out[: int(count.item())]


def _full_values(xd: torch.Tensor, b: int) -> torch.Tensor:
    from .bucketize import bucketize_device

    return bucketize_device(xd, b, [0])[0]


def _initial(xd, depth, thr, ledger) -> _DevLayer:
    n = int(xd.numel())
    vals = _full_values(xd, 1 << depth)
    record_bucketization(ledger, n, 1 << depth, [0])
    return _DevLayer(depth, _active(vals, thr), vals)


def _expand(xd, prev: _DevLayer, thr, ledger) -> _DevLayer:
    n = int(xd.numel())
    depth = prev.depth + 1
    b = 1 << depth
    if b > n:
        raise ValueError("layer depth exceeds log2 of the signal size")
    half = 1 << prev.depth
    cand = torch.cat([prev.active, prev.active + half])  # already ascending
    if 2 * prev.m_d <= depth:
        vals = torch.empty(cand.numel(), dtype=torch.complex128, device=xd.device)
        if cand.numel():
            _lib.check(
                _lib.load().afft_selective_sums(xd.data_ptr(), _device.dtype_code(xd), n, b,
                                                cand.data_ptr(), cand.numel(), vals.data_ptr(),
                                                _device.stream_ptr()),
                "selective_sums",
            )
        if ledger is not None:
            for _ in range(int(cand.numel())):
                record_bucketization(ledger, n, b, [0])
        act = _active(vals, thr, cand) if cand.numel() else cand
        return _DevLayer(depth, act, vals, cand)
    vals = _full_values(xd, b)
    record_bucketization(ledger, n, b, [0])
    return _DevLayer(depth, _active(vals, thr), vals)


@functools.lru_cache(maxsize=256)
def _search_plan(n: int, seed: int) -> SearchPlan:
    """The noisy plan of _classify_active (dsfft.py:142-150).  Deterministic in
    (n, seed), so cached: a batch decoded with one seed draws it once."""
    c = int(np.ceil(np.log2(n)))
    m = max(2, int(np.ceil(np.log2(n) ** (1.0 / 3.0))))
    rng = np.random.default_rng(seed)
    return SearchPlan(c=c, m=m, anchors=[int(t) for t in rng.integers(0, n, size=c)],
                      weights=kay_weights(m))


def _dt3_shift_table(n: int, config: DsfftConfig):
    """The DT3 fallback's random shifts (dsfft.py:207-212) for every possible stop depth d:
    p = max(12, ceil(a_m log10 max(n/2^d, 10))) draws of default_rng(seed).choice.
    Cached on (n, a_m, seed); the arrays are read-only."""
    return _dt3_shift_table_cached(n, int(config.a_m), int(config.seed))


@functools.lru_cache(maxsize=256)
def _dt3_shift_table_cached(n: int, a_m: int, seed: int):
    config = DsfftConfig(a_m=a_m, seed=seed)
    max_depth = n.bit_length() - 1
    offs, flat = [0], []
    for d in range(max_depth + 1):
        b = 1 << d
        step = n // b
        p = max(12, int(np.ceil(config.a_m * np.log10(max(step, 10)))))
        cfg = OneShotConfig(b=b, a_m=config.a_m, p=p, variant="dt3", seed=config.seed)
        try:
            cfg.validate(n)
            flat.extend(random_shifts(n, cfg))
        except ValueError:  # not reachable as a stop depth (too few samples)
            pass
        offs.append(len(flat))
    flat, offs = np.asarray(flat, dtype=np.int64), np.asarray(offs, dtype=np.int32)
    flat.setflags(write=False)
    offs.setflags(write=False)
    return flat, offs


def _replay(trace_rec, n, config, plan, dt_table, ledger, trace):
    """Ledger records and the Python trace from the native trace records."""
    if ledger is None and trace is None:
        return  # nothing to replay (the common batch case: no per-record Python work)
    flat, offs = dt_table
    for kind, depth, a, c in trace_rec:
        b = 1 << depth
        if kind in (0, 1):
            record_bucketization(ledger, n, b, [0])
        elif kind == 2:
            for _ in range(c if c >= 0 else 1):
                record_bucketization(ledger, n, b, [0])
            if trace is not None:
                trace.append(["expand", depth, a])
        elif kind == 3:
            if trace is not None:
                trace.append(["classify", depth, a, c])
        elif kind == 4:
            rsh = flat[offs[depth]:offs[depth + 1]].tolist()
            record_bucketization(ledger, n, b, structured_shifts(config.a_m) + rsh)
        elif kind == 5:
            record_bucketization(ledger, n, b, [0, 1, 2] if c == 0 else plan.shifts)


def dsfft_device(xd: torch.Tensor, k: int, config: DsfftConfig,
                 ledger: SampleLedger | None = None, trace: list | None = None
                 ) -> dict[int, complex]:
    """dsfft body (dsfft.py:250-266) for one device signal; returns the entries dict
    in the reference's insertion order (see _dsfft_arrays)."""
    pos, val = _dsfft_arrays(xd, k, config, ledger, trace)
    return _lib.entries_dict(pos, val)


def _dsfft_arrays(xd: torch.Tensor, k: int, config: DsfftConfig,
                  ledger: SampleLedger | None = None, trace: list | None = None):
    """dsfft body (dsfft.py:250-266) for one device signal: (positions, values) of the
    entries dict in insertion order.

    The layer loop runs natively (afft_dsfft, csrc/dsfft_host.cu); this wrapper draws
    the numpy-PCG64 inputs it needs (search-plan anchors, DT3 random shifts per stop
    depth), then replays the ledger and the optional ``trace`` (["expand", depth, m_d]
    / ["classify", depth, #single, #multi] in the reference's order)."""
    n = int(xd.numel())
    xd = xd.contiguous()
    noisy = config.mode != "exact"
    plan = _search_plan(n, config.seed) if noisy else None
    dt_table = _dt3_shift_table(n, config)
    anchors = np.asarray(plan.anchors if noisy else [0], dtype=np.int64)
    weights = np.asarray(plan.weights if noisy else [0.0], dtype=np.float64)
    prm = _lib.DsfftParams(
        theta=float(config.theta), mode=1 if noisy else 0, a_m=int(config.a_m),
        noise_std=float(config.noise_std), activity_floor=float(config.activity_floor),
        c=int(plan.c) if noisy else 0, m=int(plan.m) if noisy else 0,
        anchors=anchors.ctypes.data, weights=weights.ctypes.data,
        dt_shifts=dt_table[0].ctypes.data if dt_table[0].size else None,
        dt_shift_off=dt_table[1].ctypes.data,
        # a requested trace carries the reference's per-layer counts: classify every
        # layer in full; otherwise intermediate layers classify probe sets (same output)
        full_classify=int(trace is not None or os.environ.get("AFFT_DSFFT_LAZY") == "0"))
    lib = _lib.load()
    cap = max(8 * k, 1024)
    tcap = 4 * (n.bit_length() + 8)
    while True:
        pos = np.empty(cap, dtype=np.int64)
        val = np.empty(cap, dtype=np.complex128)
        cnt = ctypes.c_int64(0)
        tr = np.empty((tcap, 4), dtype=np.int32)
        tlen = ctypes.c_int32(0)
        rc = lib.afft_dsfft(xd.data_ptr(), _device.dtype_code(xd), n, int(k), ctypes.byref(prm),
                            pos.ctypes.data, val.ctypes.data, cap, ctypes.byref(cnt),
                            tr.ctypes.data, tcap, ctypes.byref(tlen), _device.stream_ptr())
        if rc == _lib.AFFT_ENOMEM and cnt.value > cap:
            cap = int(cnt.value)
            continue
        if rc == _lib.AFFT_OK and tlen.value > tcap:
            tcap = int(tlen.value)  # trace truncated: rerun with room (rare)
            continue
        _lib.check(rc, "dsfft")
        break
    _replay(tr[: tlen.value].tolist(), n, config, plan, dt_table, ledger, trace)
    m = int(cnt.value)
    return pos[:m], val[:m]


def dsfft(x, k: int, config: DsfftConfig | None = None,
          ledger: SampleLedger | None = None) -> SparseSpectrum:
    """Binary-tree sparse transform for power-of-two sizes (dsfft.py:244-267)."""
    n = _device.signal_length(x)
    if n & (n - 1):
        raise UnsupportedSizeError(f"binary-tree search needs a power-of-two size, got {n}")
    if k <= 0:
        return SparseSpectrum(n, {})
    if k > 64:
        warnings.warn(f"binary-tree search degrades for large sparsity (k={k})", stacklevel=2)
    pos, val = _dsfft_arrays(_device.as_device_signal(x), k, config or DsfftConfig(), ledger)
    return _top_k(n, k, pos, val)


_POOL_LOCK = __import__("threading").Lock()
_POOLS: dict = {}


def _worker_pool(workers: int, device):
    """A persistent thread pool per (size, device) whose threads keep their own CUDA
    stream: a worker's first decode pays the thread's and stream's set-up (measured
    ~2x a warm decode), so pools are not torn down between calls."""
    from concurrent.futures import ThreadPoolExecutor

    key = (workers, str(device))
    with _POOL_LOCK:
        pool = _POOLS.get(key)
        if pool is None:
            pool = ThreadPoolExecutor(max_workers=workers, thread_name_prefix="afft-dsfft")
            _POOLS[key] = pool
    return pool


def _dsfft_batch_native(xd: torch.Tensor, k: int, cfgs, idx: list[int]):
    """afft_dsfft_batch over the signals idx of xd (lockstep layers); returns
    {i: (positions, values)} for the signals it decoded (the others fell back)."""
    n = int(xd.shape[1])
    S = len(idx)
    plans, tables, keep = [], [], []
    prms = (_lib.DsfftParams * S)()
    for q, i in enumerate(idx):
        c = cfgs[i]
        plan = _search_plan(n, c.seed)
        table = _dt3_shift_table(n, c)
        anchors = np.asarray(plan.anchors, dtype=np.int64)
        weights = np.asarray(plan.weights, dtype=np.float64)
        keep += [anchors, weights, table]
        plans.append(plan)
        prms[q] = _lib.DsfftParams(
            theta=float(c.theta), mode=1, a_m=int(c.a_m), noise_std=float(c.noise_std),
            activity_floor=float(c.activity_floor), c=int(plan.c), m=int(plan.m),
            anchors=anchors.ctypes.data, weights=weights.ctypes.data,
            dt_shifts=table[0].ctypes.data if table[0].size else None,
            dt_shift_off=table[1].ctypes.data,
            full_classify=int(os.environ.get("AFFT_DSFFT_LAZY") == "0"))
    if idx == list(range(idx[0], idx[0] + S)):
        sub = xd[idx[0]:idx[0] + S]  # a run of signals: a view, no copy of n-sized rows
    else:
        sub = xd[idx]
    if sub.stride(-1) != 1:
        sub = sub.contiguous()
    lib = _lib.load()
    cap = max(8 * k, 1024)
    tcap = 4 * (n.bit_length() + 8)
    pos = np.empty((S, cap), dtype=np.int64)
    val = np.empty((S, cap), dtype=np.complex128)
    cnt = np.zeros(S, dtype=np.int64)
    tr = np.empty((S, tcap, 4), dtype=np.int32)
    tlen = np.zeros(S, dtype=np.int32)
    fb = np.zeros(S, dtype=np.int32)
    _lib.check(lib.afft_dsfft_batch(
        sub.data_ptr(), _device.dtype_code(sub), n, S, int(sub.stride(0)), int(k), prms,
        pos.ctypes.data, val.ctypes.data, cap, cnt.ctypes.data, tr.ctypes.data, tcap,
        tlen.ctypes.data, fb.ctypes.data, _device.stream_ptr()), "dsfft_batch")
    out = {}
    for q, i in enumerate(idx):
        if fb[q] or tlen[q] > tcap:
            continue
        m = int(cnt[q])
        out[i] = (pos[q, :m], val[q, :m])
    return out


def _top_k_arrays(k: int, pos, val):
    """truncate_spectrum (oneshot.py:260-263): the k largest |v|, ties to the smaller
    position, in that order (the keys are distinct, so the sort is total).  The sort runs
    in afft_truncate_host with the GIL released (worker threads overlap it)."""
    pos = np.ascontiguousarray(pos, dtype=np.int64)
    val = np.ascontiguousarray(val, dtype=np.complex128)
    m = min(int(pos.size), int(k))
    op = np.empty(max(m, 1), dtype=np.int64)
    ov = np.empty(max(m, 1), dtype=np.complex128)
    cnt = ctypes.c_int64(0)
    _lib.check(_lib.load().afft_truncate_host(pos.ctypes.data, val.ctypes.data, int(pos.size),
                                              int(k), op.ctypes.data, ov.ctypes.data,
                                              ctypes.byref(cnt)), "truncate")
    m = int(cnt.value)
    return op[:m], ov[:m]


def _top_k(n: int, k: int, pos, val) -> SparseSpectrum:
    """truncate_spectrum as the drop-in result type."""
    op, ov = _top_k_arrays(k, pos, val)
    return SparseSpectrum._trusted(n, _lib.entries_dict(op, ov))


def _guided_parts(items: list[int], workers: int, cap: int) -> list[list[int]]:
    """Chunks of shrinking size (guided scheduling): ceil(remaining / (1.5 workers))
    signals each, at most ``cap``, at least 1 — long lockstep chunks first, single signals
    last, so the workers do not all finish at once and the caller's per-signal result
    work (the entries dicts) has only a short tail after the last kernels."""
    parts, at = [], 0
    while at < len(items):
        left = len(items) - at
        size = max(1, min(int(cap), -(-2 * left // (3 * max(1, workers)))))
        parts.append(items[at:at + size])
        at += size
    return parts


def dsfft_batch(xs, k: int, configs, streams: int = 8, lockstep: bool | None = None,
                chunk: int = 4, guided: bool = True) -> list[SparseSpectrum]:
    """DSFFT over several signals, in input order.

    ``lockstep`` (the default for two or more signals): noisy decodes of large
    power-of-two signals with a given noise level run in lockstep (afft_dsfft_batch: up to
    ``chunk`` signals per call, one launch per layer step for all of them; the chunks on
    up to ``streams`` worker streams, sized by `_guided_parts` unless ``guided=False``);
    the workers return the truncated (positions, values) arrays and the calling thread
    builds each SparseSpectrum's dict while they run their next chunk.  Signals that leave
    the common path, exact-mode signals and ``lockstep=False`` take the per-signal native
    loop, one signal per worker stream (_dsfft_batch_threads).  All forms give identical
    results (tests/test_gpu_dsfft_batch.py).  Measured at config 4 (32 signals, 20 dB,
    tools/dsfft_api_sweep.py, tools/dsfft_lockstep_sweep.py): per-signal loops 1.35 k
    signals/s; lockstep with the dicts built by the workers 1.27-1.34 k (every worker
    finishes at once and the dicts, ~0.2 ms of GIL time each, form a serial tail); with the
    dicts on the calling thread and 2 signals per call 1.53 k; the C ABI alone (arrays, no
    dicts) 2.0-2.1 k on 8 streams x 4 signals."""
    xd0 = _device.as_device_batch(xs)
    count0 = int(xd0.shape[0])
    cfgs0 = [configs[i] if isinstance(configs, (list, tuple)) else configs for i in range(count0)]
    n0 = int(xd0.shape[1]) if count0 else 0
    done: dict[int, SparseSpectrum] = {}
    if lockstep is None:  # the lockstep form is the faster one for batches (bench: c4dsfft)
        lockstep = count0 >= 2
    if lockstep and count0 and n0 >= (1 << 16) and not (n0 & (n0 - 1)):
        cand = [i for i in range(count0) if cfgs0[i].mode != "exact" and cfgs0[i].noise_std > 0]
        size = max(1, int(chunk))
        if guided:
            parts = _guided_parts(cand, max(1, min(int(streams), len(cand))), size)
        else:
            parts = [cand[c0:c0 + size] for c0 in range(0, len(cand), size)]
        def chunk_fn(part):  # the host-side truncation overlaps other chunks' kernels
            return {i: _top_k_arrays(k, p, v)
                    for i, (p, v) in _dsfft_batch_native(xd0, k, cfgs0, part).items()}

        def to_spectra(res):
            # on the caller's thread, as each chunk arrives: the 4096-entry dicts need the
            # GIL (~0.2 ms per signal); the workers are already inside their next chunk's
            # native call (GIL released), so only the last chunks' dicts are a tail
            for i, (op, ov) in res.items():
                done[i] = SparseSpectrum._trusted(n0, _lib.entries_dict(op, ov))

        _on_worker_streams(xd0, parts, streams, chunk_fn, consume=to_spectra)
    rest = [i for i in range(count0) if i not in done]
    if rest:
        outs = _dsfft_batch_threads(xd0[rest] if len(rest) < count0 else xd0, k,
                                    [cfgs0[i] for i in rest], streams)
        for i, o in zip(rest, outs):
            done[i] = o
    return [done[i] for i in range(count0)]


def _on_worker_streams(xd: torch.Tensor, items, streams: int, fn, consume=None):
    """fn(item) for every item, on up to `streams` persistent worker threads with their
    own CUDA streams (ordered after the caller's stream, joined back into it).  With
    ``consume``, each result is passed to it on the calling thread as soon as it (and
    every earlier item's) is ready, while the workers carry on."""
    import threading

    take = consume if consume is not None else (lambda r: r)
    workers = max(1, min(int(streams), len(items)))
    if workers <= 1:
        return [take(fn(it)) for it in items]
    main = torch.cuda.current_stream(xd.device)
    ready = torch.cuda.Event()
    ready.record(main)
    done = []
    lock = threading.Lock()
    local = _worker_local

    def work(it):
        st = getattr(local, "stream", None)
        if st is None or st.device != xd.device:
            st = local.stream = torch.cuda.Stream(device=xd.device)
        st.wait_event(ready)
        with torch.cuda.stream(st):
            out = fn(it)
            ev = torch.cuda.Event()
            ev.record(st)
        with lock:
            done.append(ev)
        return out

    out = [take(r) for r in _worker_pool(workers, xd.device).map(work, items)]
    for ev in done:
        main.wait_event(ev)
    return out


def _dsfft_batch_threads(xs, k: int, configs, streams: int = 8) -> list[SparseSpectrum]:
    """DSFFT over several signals, in input order.  Each signal's layer loop is
    data-dependent (one read-back per layer), so one signal alone leaves the GPU idle
    during its read-backs; with streams > 1 signals run on worker threads, each with
    its own CUDA stream (the library is reentrant per stream and the native loop runs
    without the GIL), overlapping one signal's read-backs with another's kernels.
    Results are identical to the sequential run; 8 streams measured best at config 4
    (tools/dsfft_streams.py: 1 / 2 / 4 / 8 streams 246 / 368 / 490 / 531 signals/s,
    the GPU 94% busy at 8, tools/dsfft_gpu_busy.py)."""
    import threading

    xd = _device.as_device_batch(xs)
    count = int(xd.shape[0])
    cfgs = [configs[i] if isinstance(configs, (list, tuple)) else configs for i in range(count)]
    workers = max(1, min(int(streams), count))
    if workers == 1:
        return [dsfft(xd[i], k, cfgs[i]) for i in range(count)]
    main = torch.cuda.current_stream(xd.device)
    ready = torch.cuda.Event()
    ready.record(main)  # the batch was produced on the caller's stream
    done = []
    lock = threading.Lock()
    local = _worker_local

    def work(i):
        st = getattr(local, "stream", None)
        if st is None or st.device != xd.device:
            st = local.stream = torch.cuda.Stream(device=xd.device)
        st.wait_event(ready)
        with torch.cuda.stream(st):
            out = dsfft(xd[i], k, cfgs[i])
            ev = torch.cuda.Event()
            ev.record(st)
        with lock:
            done.append(ev)
        return out

    out = list(_worker_pool(workers, xd.device).map(work, range(count)))
    for ev in done:
        main.wait_event(ev)
    return out


_worker_local = __import__("threading").local()


def _to_tree_layer(layer: _DevLayer) -> TreeLayer:
    if layer.cand is None:
        vals = layer.values.cpu().numpy()
        values = {i: complex(v) for i, v in enumerate(vals)}
    else:
        vals = layer.values.cpu().numpy()
        values = {int(i): complex(v) for i, v in zip(layer.cand.cpu().numpy(), vals)}
    return TreeLayer(depth=layer.depth, values=values,
                     active=set(int(i) for i in layer.active.cpu().numpy()))


def initial_layer(x, depth: int, ledger: SampleLedger | None, threshold: float) -> TreeLayer:
    """Full size-2^depth bucketization at shift 0 plus its active set (dsfft.py:73-79)."""
    xd = _device.as_device_signal(x)
    return _to_tree_layer(_initial(xd, depth, threshold, ledger))


def expand_layer(x, prev: TreeLayer, ledger: SampleLedger | None, threshold: float) -> TreeLayer:
    """Next layer, selectively when few buckets are active (dsfft.py:82-115)."""
    xd = _device.as_device_signal(x)
    act = torch.tensor(sorted(prev.active), dtype=torch.int64, device=xd.device)
    return _to_tree_layer(_expand(xd, _DevLayer(prev.depth, act), threshold, ledger))


def non_aliasing_probability(n: int, k: int, b: int) -> float:
    """P(k uniform distinct tones land in k distinct buckets) (dsfft.py:270-285); scalar formula."""
    if b < 1 or n % b:
        raise ValueError(f"bucket count {b} does not divide {n}")
    if not 1 <= k <= n:
        raise ValueError(f"need 1 <= k <= n, got k={k}")
    if k > b:
        return 0.0
    step = n // b
    prob = 1.0
    for j in range(1, k):
        prob *= (n - j * step) / (n - j)
    return prob


def non_aliasing_probability_limit(k: int, b: int) -> float:
    """Large-n limit prod_{j<k} (1 - j/b) (dsfft.py:288-297); scalar formula."""
    if k < 1 or b < 1:
        raise ValueError("k and b must be positive")
    if k > b:
        return 0.0
    prob = 1.0
    for j in range(1, k):
        prob *= 1.0 - j / b
    return prob


__all__ = ["DsfftConfig", "TreeLayer", "dsfft", "dsfft_batch", "expand_layer", "initial_layer",
           "non_aliasing_probability", "non_aliasing_probability_limit", "gather_indices"]
