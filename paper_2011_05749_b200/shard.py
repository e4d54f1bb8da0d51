"""Signal-parallel sharding across ranks.

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


def max_over_ranks(values: list[float], device, group=None) -> list[float]:
    """Element-wise max over ranks (timings are reported as the slowest rank)."""
    t = torch.tensor(values, dtype=torch.float64, device=device)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return [float(v) for v in t.tolist()]
