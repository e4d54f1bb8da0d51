"""Signal-parallel sharding across ranks, and the one-huge-signal
R-FFAST split (the §8(e) stretch row, `SearchShard`).

Every algorithm on the path is independent per signal, so a batch is split into
contiguous per-rank slices with no data-path collective; the only exchange is
the final gather of the fixed-size result slots ([signals, k] positions and
values plus per-signal counts) — one all-gather over NCCL/NVLink on GPUs, gloo
in the CPU tests.  Ranks hold equal slices (the batch is padded to a multiple
of the world size by the caller if needed).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """[start, stop) of rank's contiguous slice; equal slices, the first total % world get +1."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def gather_slots(pos: torch.Tensor, val: torch.Tensor, count: torch.Tensor, group=None):
    """All-gather equal-size per-rank result slots into [world * signals, ...] tensors.

    pos [s, k] int64, val [s, k] complex128 (sent as a float64 view), count [s] int32.
    """
    world = dist.get_world_size(group)
    if world == 1:
        return pos, val, count
    if pos.is_cuda and dist.get_backend(group) == "gloo":
        # a gloo group over device results (tests on one GPU): stage through the host
        dev = pos.device
        return tuple(t.to(dev) for t in gather_slots(pos.cpu(), val.cpu(), count.cpu(), group))
    vr = torch.view_as_real(val.contiguous())
    out_pos = torch.empty((world * pos.shape[0],) + tuple(pos.shape[1:]), dtype=pos.dtype,
                          device=pos.device)
    out_val = torch.empty((world * vr.shape[0],) + tuple(vr.shape[1:]), dtype=vr.dtype,
                          device=vr.device)
    out_cnt = torch.empty(world * count.shape[0], dtype=count.dtype, device=count.device)
    dist.all_gather_into_tensor(out_pos, pos.contiguous(), group=group)
    dist.all_gather_into_tensor(out_val, vr, group=group)
    dist.all_gather_into_tensor(out_cnt, count.contiguous(), group=group)
    return out_pos, torch.view_as_complex(out_val), out_cnt


def sharded_batch(decode, total: int, group=None):
    """Run ``decode(start, stop) -> (pos [s, k] int64, val [s, k] complex128,
    count [s] int32)`` on this rank's contiguous slice of ``total`` independent signals
    and return every rank's slots, in signal order, on every rank (no
    data-path collective, one all-gather of the fixed result slots).  Slices that differ
    by one signal are padded to the longest before the gather and the pad rows dropped
    after it.  Without an initialised process group this is ``decode(0, total)``."""
    if not (dist.is_available() and dist.is_initialized()):
        return decode(0, total)
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    start, stop = shard_range(total, rank, world)
    pos, val, count = decode(start, stop)
    if world == 1:
        return pos, val, count
    per = -(-total // world)
    pad = per - (stop - start)
    if pad:
        pos = torch.cat([pos, pos.new_zeros((pad,) + tuple(pos.shape[1:]))])
        val = torch.cat([val, val.new_zeros((pad,) + tuple(val.shape[1:]))])
        count = torch.cat([count, count.new_zeros(pad)])
    gp, gv, gc = gather_slots(pos, val, count, group)
    if total % world == 0:
        return gp, gv, gc
    keep = torch.cat([torch.arange(r * per, r * per + b - a, device=gp.device)
                      for r in range(world) for a, b in [shard_range(total, r, world)]])
    return gp[keep], gv[keep], gc[keep]


def _slice(seq, a, b):
    """Per-signal arguments: a list/tuple is sliced with the signals, anything else is
    shared by every signal."""
    return seq[a:b] if isinstance(seq, (list, tuple)) else seq


def ffast_sharded(x, k: int, factors, group=None, **kw):
    """`ffast_batch` (configs 1 and 5) over this rank's slice of the (signals, n) block
    x; the top-k slots of all signals on every rank."""
    from .batch import ffast_batch

    def decode(a, b):
        r = ffast_batch(x[a:b], k, factors, **kw)
        return r.pos, r.val, r.count

    return sharded_batch(decode, len(x), group)


def rffast_sharded(x, k: int, factors, search, group=None, **kw):
    """`rffast_batch` (config 3) signal-sharded: ``search`` is one SearchPlan or a list
    with one per signal (sliced with the signals)."""
    from .rffast import rffast_batch

    def decode(a, b):
        r = rffast_batch(x[a:b], k, factors, _slice(search, a, b), **kw)
        return r.pos, r.val, r.count

    return sharded_batch(decode, len(x), group)


def sfft_dt_sharded(x, k: int, b: int, a_m: int = 4, p: int = 12, variant: str = "dt3",
                    seeds=None, group=None):
    """`sfft_dt_batch` (configs 2 and 4) signal-sharded with per-signal seeds."""
    from .oneshot import sfft_dt_batch

    def decode(a, e):
        r = sfft_dt_batch(x[a:e], k, b, a_m, p, variant,
                          seeds=None if seeds is None else list(seeds)[a:e])
        return r.pos, r.val, r.count

    return sharded_batch(decode, len(x), group)


def spectra_to_slots(spectra, k: int, device=None):
    """list[SparseSpectrum] -> ([s, k] positions, [s, k] values, [s] counts) in each
    spectrum's insertion order (the fixed-size slots `gather_slots` exchanges)."""
    import numpy as np

    s = len(spectra)
    pos = np.zeros((s, k), dtype=np.int64)
    val = np.zeros((s, k), dtype=np.complex128)
    cnt = np.zeros(s, dtype=np.int32)
    for i, sp in enumerate(spectra):
        m = min(len(sp.entries), k)
        cnt[i] = m
        if m:
            pos[i, :m] = np.fromiter(sp.entries.keys(), dtype=np.int64, count=len(sp.entries))[:m]
            val[i, :m] = np.fromiter(sp.entries.values(), dtype=np.complex128,
                                     count=len(sp.entries))[:m]
    return tuple(torch.from_numpy(t).to(device) if device is not None else torch.from_numpy(t)
                 for t in (pos, val, cnt))


def dsfft_sharded(x, k: int, configs, group=None, **kw):
    """`dsfft_batch` (config 4) signal-sharded; ``configs`` is one DsfftConfig or a list
    with one per signal.  The per-signal spectra become fixed [s, k] slots on x's device
    (NCCL gathers device tensors) before the gather."""
    from .dsfft import dsfft_batch

    device = x.device if isinstance(x, torch.Tensor) else None

    def decode(a, b):
        return spectra_to_slots(dsfft_batch(x[a:b], k, _slice(configs, a, b), **kw), k, device)

    return sharded_batch(decode, len(x), group)


def max_over_ranks(values: list[float], device, group=None) -> list[float]:
    """Element-wise max over ranks (timings are reported as the slowest rank)."""
    t = torch.tensor(values, dtype=torch.float64, device=device)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return [float(v) for v in t.tolist()]


class SearchShard:
    """Split of one R-FFAST decode's singleton search over `world` ranks (SURVEY §8(e),
    stretch row: "node x candidate-range split of the singleton search, MINLOC
    all-reduce per peeling round").

    Every rank builds the same graph and runs the same peeling rounds; rank r scans
    the candidate chunks ch = r (mod world) of every active node, and once per round
    `reduce_min(scores, cands)` must make both device tensors (float64 / int32, the
    per-(node, chunk) partial minima, unscanned slots +inf / INT32_MAX) their
    element-wise minimum over the ranks, in place.  Exactly one rank holds a real
    value per slot, so MIN over each array is the MINLOC; results equal the
    single-rank decode bit for bit.
    """

    def __init__(self, rank: int, world: int, reduce_min):
        if world < 1 or not 0 <= rank < world:
            raise ValueError(f"bad rank {rank} / world {world}")
        self.rank, self.world, self.reduce_min = int(rank), int(world), reduce_min

    @classmethod
    def from_process_group(cls, group=None) -> "SearchShard":
        """NCCL (or gloo) all-reduce MIN over a torch.distributed group."""
        def reduce_min(scores: torch.Tensor, cands: torch.Tensor) -> None:
            dist.all_reduce(scores, op=dist.ReduceOp.MIN, group=group)
            dist.all_reduce(cands, op=dist.ReduceOp.MIN, group=group)

        return cls(dist.get_rank(group), dist.get_world_size(group), reduce_min)
