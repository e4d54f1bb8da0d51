"""Deterministic binary-tree search (DSFFT) on the GPU.

Drop-in for /root/reference/pkg/src/aliasfft/dsfft.py.  The layer loop is
host control flow (one small count read per layer); every layer's data stays on
the device: full layers are size-2^d bucketizations (one-CTA or four-step
DFT), selective layers are direct alias sums, activity is a device stream
compaction, classification reuses the exact / noisy singleton kernels on
measurement rows built with coset reuse (csrc/dsfft.cu), and leftover aliased
buckets go through the sFFT-DT3 kernels.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass, field, replace

import numpy as np
import torch

from . import _device, _lib
from .bucketize import SampleLedger, gather_indices, record_bucketization
from .oneshot import OneShotConfig, random_shifts, structured_shifts
from .peeling import (
    STATE_CODE,
    NodeState,
    SearchPlan,
    UnsupportedSizeError,
    exact_thresholds_device,
    kay_weights,
)
from .signals import SparseSpectrum

STATE_SINGLE = STATE_CODE[NodeState.SINGLE_TON]
STATE_MULTI = STATE_CODE[NodeState.MULTI_TON]


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


def _threshold(config: DsfftConfig, depth: int) -> float:
    return max(config.activity_floor, 3.0 * config.noise_std / np.sqrt(1 << depth))


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


# Deep layers (n/b <= 32) read the signal's normalised spectrum Y = fft(x)/n, computed
# once per dsfft_device call, through the alias identity (afft_alias_rows) instead of
# running min(#shifts, n/b) size-b DFTs over the whole signal at every layer.
_ALIAS_MAX_L = 32
_SPECTRA: dict[tuple, list] = {}  # (data_ptr, numel) -> [Y or None, ||Y||^2 or None]


def _spectrum(xd: torch.Tensor):
    """[Y, ||Y||^2] for a signal registered by dsfft_device, else None."""
    ent = _SPECTRA.get((xd.data_ptr(), xd.numel()))
    if ent is None:
        return None
    if ent[0] is None:
        from .bucketize import bucketize_device

        ent[0] = bucketize_device(xd, int(xd.numel()), [0])[0]
    return ent


def _alias_ok(xd: torch.Tensor, b: int) -> bool:
    return int(xd.numel()) // b <= _ALIAS_MAX_L and (xd.data_ptr(), xd.numel()) in _SPECTRA


def _full_values(xd: torch.Tensor, b: int) -> torch.Tensor:
    if _alias_ok(xd, b):
        Y = _spectrum(xd)[0]
        vals = torch.empty(b, dtype=torch.complex128, device=xd.device)
        _lib.check(_lib.load().afft_alias_rows(Y.data_ptr(), int(xd.numel()), b, None, 0, None, 0,
                                               None, None, vals.data_ptr(), _device.stream_ptr()),
                   "alias_rows")
        return vals
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


def _rows(xd, b, shifts, idx, energy=False):
    n = int(xd.numel())
    rows = torch.empty((max(1, idx.numel()), len(shifts)), dtype=torch.complex128,
                       device=xd.device)
    en = torch.empty(b, dtype=torch.float64, device=xd.device) if energy else None
    sb, ns = _lib.host_i64(shifts)
    if _alias_ok(xd, b):
        Y = _spectrum(xd)[0]
        _lib.check(
            _lib.load().afft_alias_rows(Y.data_ptr(), n, b, sb, ns,
                                        idx.data_ptr() if idx.numel() else None, idx.numel(),
                                        rows.data_ptr(), None if en is None else en.data_ptr(),
                                        None, _device.stream_ptr()),
            "alias_rows",
        )
        return rows[: idx.numel()], en
    _lib.check(
        _lib.load().afft_bucketize_rows(xd.data_ptr(), _device.dtype_code(xd), n, b, sb, ns,
                                        idx.data_ptr() if idx.numel() else None, idx.numel(),
                                        rows.data_ptr(), None if en is None else en.data_ptr(),
                                        _device.stream_ptr()),
        "bucketize_rows",
    )
    return rows[: idx.numel()], en


def _search_plan(n: int, seed: int) -> SearchPlan:
    """The noisy plan of _classify_active (dsfft.py:142-150)."""
    c = int(np.ceil(np.log2(n)))
    m = max(2, int(np.ceil(np.log2(n) ** (1.0 / 3.0))))
    rng = np.random.default_rng(seed)
    return SearchPlan(c=c, m=m, anchors=[int(t) for t in rng.integers(0, n, size=c)],
                      weights=kay_weights(m))


def _classify(xd, layer: _DevLayer, config: DsfftConfig, ledger):
    """_classify_active (dsfft.py:118-174): decoded single-tons and multi-ton buckets."""
    n = int(xd.numel())
    b = layer.b
    lib = _lib.load()
    sp = _device.stream_ptr()
    act = layer.active
    A = int(act.numel())
    entries: dict[int, complex] = {}
    multitons: list[int] = []
    if config.mode == "exact":
        shifts = [0, 1, 2]
        record_bucketization(ledger, n, b, shifts)
        if A == 0:
            return entries, multitons
        rows, _ = _rows(xd, b, shifts, act)
        eps = float(exact_thresholds_device(xd).item())
        st = torch.empty(A, dtype=torch.int8, device=xd.device)
        f0 = torch.full((A,), -1, dtype=torch.int64, device=xd.device)
        val = torch.zeros(A, dtype=torch.complex128, device=xd.device)
        _lib.check(lib.afft_classify_exact(rows.data_ptr(), act.data_ptr(), A, b, n, eps, eps,
                                           st.data_ptr(), f0.data_ptr(), val.data_ptr(), sp),
                   "classify_exact")
    else:
        plan = _search_plan(n, config.seed)
        shifts = plan.shifts
        record_bucketization(ledger, n, b, shifts)
        R = len(shifts)
        base = config.noise_std / np.sqrt(b) * np.sqrt(R)
        # the floor 1e-8 sqrt(max energy) only matters above 1.5 base; with the
        # spectrum resident, max energy <= R (n/b) ||Y||^2 bounds it without the
        # all-bucket energy pass (thresholds identical either way)
        skip = False
        if config.noise_std > 0.0 and _alias_ok(xd, b):
            ent = _spectrum(xd)
            if ent[1] is None:
                ent[1] = float((ent[0].abs() ** 2).sum().item())
            skip = 1e-8 * np.sqrt(R * (n // b) * ent[1]) < 1.5 * base
        rows, energy = _rows(xd, b, shifts, act, energy=not skip)
        if config.noise_std > 0.0:
            floor = 0.0 if skip else 1e-8 * np.sqrt(float(energy.max().item()))
            t0, t1 = max(1.5 * base, floor), max(2.5 * base, floor)
        else:
            from .rffast import robust_thresholds_device

            quiet = torch.ones(b, dtype=torch.uint8, device=xd.device)
            if A:
                quiet[act] = 0
            a0, a1 = robust_thresholds_device(energy.unsqueeze(0), R, quiet.unsqueeze(0))
            t0, t1 = float(a0.item()), float(a1.item())
        if A == 0:
            return entries, multitons
        st = torch.empty(A, dtype=torch.int8, device=xd.device)
        f0 = torch.full((A,), -1, dtype=torch.int64, device=xd.device)
        val = torch.zeros(A, dtype=torch.complex128, device=xd.device)
        rn = torch.empty(A, dtype=torch.float64, device=xd.device)
        need = int(lib.afft_singleton_workspace_size(n, A, b, plan.c, plan.m))
        ws = torch.empty(need, dtype=torch.uint8, device=xd.device)
        sb, ns = _lib.host_i64(shifts)
        wb = _lib.host_f64(plan.weights.tolist())
        _lib.check(lib.afft_classify_noisy(rows.data_ptr(), act.data_ptr(), A, b, n, sb, ns,
                                           plan.c, plan.m, wb, float(t0), float(t1),
                                           st.data_ptr(), f0.data_ptr(), val.data_ptr(),
                                           rn.data_ptr(), ws.data_ptr(), ws.numel(), sp),
                   "classify_noisy")
    # one synchronisation for the four result arrays (pinned, non-blocking copies)
    host = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in (st, f0, val, act)]
    for h, t in zip(host, (st, f0, val, act)):
        h.copy_(t, non_blocking=True)
    torch.cuda.current_stream(xd.device).synchronize()
    st_h, f0_h, val_h, act_h = (h.numpy() for h in host)
    single = st_h == STATE_SINGLE
    multi = st_h == STATE_MULTI
    # entries in ascending-bucket order, as the reference inserts them
    entries.update(zip(f0_h[single].tolist(), val_h[single].tolist()))
    multitons.extend(act_h[multi].tolist())
    return entries, multitons


def _resolve_aliased(xd, b, buckets, k_remaining, config, ledger):
    """Pencil + pursuit for buckets still holding several tones (dsfft.py:201-228)."""
    n = int(xd.numel())
    step = n // b
    p = max(12, int(np.ceil(config.a_m * np.log10(max(step, 10)))))
    cfg = OneShotConfig(b=b, a_m=config.a_m, p=p, variant="dt3", seed=config.seed)
    cfg.validate(n)
    rsh = random_shifts(n, cfg)
    shifts = structured_shifts(config.a_m) + rsh
    record_bucketization(ledger, n, b, shifts)
    idx = torch.tensor(buckets, dtype=torch.int64, device=xd.device)
    rows, _ = _rows(xd, b, shifts, idx)
    nm, R, a_m = len(buckets), len(shifts), config.a_m
    lib = _lib.load()
    sp = _device.stream_ptr()
    counts = torch.empty(nm, dtype=torch.int32, device=xd.device)
    sig = torch.empty((nm, a_m), dtype=torch.float64, device=xd.device)
    kk = min(k_remaining, a_m * nm)
    _lib.check(lib.afft_dt_detect(rows.data_ptr(), 1, nm, R, a_m, int(kk), counts.data_ptr(),
                                  sig.data_ptr(), sp), "detect_sparsity")
    rs = torch.tensor(rsh, dtype=torch.int64, device=xd.device)
    pos = torch.empty((nm, a_m), dtype=torch.int64, device=xd.device)
    val = torch.empty((nm, a_m), dtype=torch.complex128, device=xd.device)
    cnt = torch.empty(nm, dtype=torch.int32, device=xd.device)
    _lib.check(lib.afft_dt_solve(rows.data_ptr(), rs.data_ptr(), 1, nm, a_m, p, counts.data_ptr(),
                                 idx.data_ptr(), 3, a_m, b, n, pos.data_ptr(), val.data_ptr(),
                                 cnt.data_ptr(), sp), "dt3 solve")
    cnt_h, pos_h, val_h = cnt.cpu().numpy(), pos.cpu().numpy(), val.cpu().numpy()
    out: dict[int, complex] = {}
    for r in range(nm):
        for j in range(int(cnt_h[r])):
            out[int(pos_h[r, j])] = complex(val_h[r, j])
    return out


def _calibrate_noise_device(xd, k, ledger) -> float:
    """Time-domain noise std from one wide bucketization (dsfft.py:231-241)."""
    n = int(xd.numel())
    b = min(n, 1 << max(0, int(np.ceil(np.log2(32 * k)))))
    vals = _full_values(xd, b)
    record_bucketization(ledger, n, b, [0])
    med = torch.empty(1, dtype=torch.float64, device=xd.device)
    _lib.check(_lib.load().afft_median(vals.data_ptr(), 1, b, 1, med.data_ptr(),
                                       _device.stream_ptr()), "median")
    return float(np.sqrt(b * float(med.item()) / np.log(2.0)))


def dsfft_device(xd: torch.Tensor, k: int, config: DsfftConfig,
                 ledger: SampleLedger | None = None, trace: list | None = None
                 ) -> dict[int, complex]:
    """dsfft body (dsfft.py:250-266) for one device signal; returns the entries dict.
    ``trace`` (optional) collects ["expand", depth, m_d] / ["classify", depth, #single,
    #multi] records in the order the reference executes them."""
    key = (xd.data_ptr(), xd.numel())
    _SPECTRA[key] = [None, None]
    try:
        return _dsfft_layers(xd, k, config, ledger, trace)
    finally:
        _SPECTRA.pop(key, None)


def _dsfft_layers(xd, k, config, ledger, trace):
    n = int(xd.numel())
    max_depth = n.bit_length() - 1
    log = trace.append if trace is not None else (lambda rec: None)
    if config.mode != "exact" and config.noise_std <= 0.0:
        config = replace(config, noise_std=_calibrate_noise_device(xd, k, ledger))
    depth = min(max(0, int(np.ceil(np.log2(k)))), max_depth)
    layer = _initial(xd, depth, _threshold(config, depth), ledger)
    while layer.m_d < config.theta * k and layer.depth < max_depth:
        layer = _expand(xd, layer, _threshold(config, layer.depth + 1), ledger)
        log(["expand", layer.depth, layer.m_d])
    entries, multitons = _classify(xd, layer, config, ledger)
    log(["classify", layer.depth, len(entries), len(multitons)])
    while config.mode != "exact" and multitons and layer.depth < max_depth:
        layer = _expand(xd, layer, _threshold(config, layer.depth + 1), ledger)
        log(["expand", layer.depth, layer.m_d])
        entries, multitons = _classify(xd, layer, config, ledger)
        log(["classify", layer.depth, len(entries), len(multitons)])
    remaining = k - len(entries)
    if multitons and remaining > 0:
        entries.update(_resolve_aliased(xd, layer.b, multitons, remaining, config, ledger))
    return entries


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
    entries = dsfft_device(_device.as_device_signal(x), k, config or DsfftConfig(), ledger)
    ranked = sorted(entries.items(), key=lambda item: (-abs(item[1]), item[0]))
    return SparseSpectrum(n, dict(ranked[:k]))


def dsfft_batch(xs, k: int, configs, streams: int = 1) -> list[SparseSpectrum]:
    """DSFFT over several signals, in input order.  Each signal's layer path is
    data-dependent host control flow; with streams > 1 signals run on worker threads,
    each with its own CUDA stream (the library is reentrant per stream).  Measured at
    config 4 (tools/bench_suite.py): 4 streams are no faster than 1 — the per-layer
    host work holds the GIL — and give identical results, so the default is 1."""
    import threading
    from concurrent.futures import ThreadPoolExecutor

    xd = _device.as_device_batch(xs)
    count = int(xd.shape[0])
    cfgs = [configs[i] if isinstance(configs, (list, tuple)) else configs for i in range(count)]
    workers = max(1, min(int(streams), count))
    if workers == 1:
        return [dsfft(xd[i], k, cfgs[i]) for i in range(count)]
    main = torch.cuda.current_stream(xd.device)
    local = threading.local()
    made: list = []
    lock = threading.Lock()

    def work(i):
        if not hasattr(local, "stream"):
            local.stream = torch.cuda.Stream(device=xd.device)
            local.stream.wait_stream(main)  # the batch was produced on the caller's stream
            with lock:
                made.append(local.stream)
        with torch.cuda.stream(local.stream):
            return dsfft(xd[i], k, cfgs[i])

    with ThreadPoolExecutor(max_workers=workers) as ex:
        out = list(ex.map(work, range(count)))
    for st in made:
        main.wait_stream(st)
    return out

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
