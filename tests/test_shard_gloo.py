"""Multi-rank path of the signal-sharded bench on CPU: world_size 2 over gloo.

Checks the slice arithmetic and that the result-slot all-gather (NCCL on the GPU
box) reassembles every rank's [signals, k] slots in rank order, and that the
timing reduction is a max over ranks.
"""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2011_05749_b200.shard import gather_slots, max_over_ranks, shard_range


def test_shard_range_partitions():
    for total in (0, 1, 7, 8192, 8193):
        for world in (1, 2, 3, 8):
            spans = [shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    total, k = 10, 4
    a, b = shard_range(total, rank, world)
    sig = torch.arange(a, b)
    pos = (sig[:, None] * 100 + torch.arange(k)[None, :]).to(torch.int64)
    val = torch.complex(pos.double(), -pos.double())
    cnt = torch.full((b - a,), rank + 1, dtype=torch.int32)
    gp, gv, gc = gather_slots(pos, val, cnt)
    t = max_over_ranks([float(rank), 10.0 - rank], torch.device("cpu"))
    q.put((rank, gp.tolist(), gv.real.tolist(), gc.tolist(), t))
    dist.destroy_process_group()


def test_gather_slots_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for rank, gp, gv, gc, t in res:
        assert [row[0] // 100 for row in gp] == list(range(10))
        assert gv == [[float(v) for v in row] for row in gp]
        assert gc == [1] * 5 + [2] * 5
        assert t == [1.0, 10.0]


def _min_worker(rank, world, port, q):
    import numpy as np

    from paper_2011_05749_b200.shard import SearchShard

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sh = SearchShard.from_process_group()
    # slot i belongs to rank i % world; the others hold (+inf, INT32_MAX)
    count = 7
    scores = torch.full((count,), float("inf"), dtype=torch.float64)
    cands = torch.full((count,), 2**31 - 1, dtype=torch.int32)
    for i in range(rank, count, world):
        scores[i] = 0.5 * i + 0.25
        cands[i] = 100 + i
    sh.reduce_min(scores, cands)
    q.put((rank, sh.rank, sh.world, scores.tolist(), cands.tolist()))
    dist.destroy_process_group()


def test_search_shard_exchange_world2():
    """SearchShard.from_process_group: the per-round partial exchange (two all-reduce
    MIN, NCCL on GPUs) leaves every rank with the owner's value in every slot."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_min_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for rank, r2, w2, scores, cands in got:
        assert (r2, w2) == (rank, 2)
        assert scores == [0.5 * i + 0.25 for i in range(7)]
        assert cands == [100 + i for i in range(7)]


def _sharded_worker(rank, world, port, q):
    from paper_2011_05749_b200.shard import sharded_batch, spectra_to_slots
    from paper_2011_05749_b200 import SparseSpectrum

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = {}
    for total in (5, 6, 1):  # ragged slices, equal slices, fewer signals than ranks
        calls = []

        def decode(a, b, k=3):
            calls.append((a, b))
            # the stand-in decoder: signal i "recovers" i % 3 + 1 tones at 10 i + j
            sp = [SparseSpectrum(1000, {10 * i + j: complex(i, -j) for j in range(i % 3 + 1)})
                  for i in range(a, b)]
            return spectra_to_slots(sp, k)

        gp, gv, gc = sharded_batch(decode, total)
        out[total] = (calls, gp.tolist(), gv.real.tolist(), gv.imag.tolist(), gc.tolist())
    q.put((rank, out))
    dist.destroy_process_group()


def test_sharded_batch_world2():
    """The C2/C3/C4 signal-sharded harness: every rank decodes only its slice and ends
    with all signals' slots in signal order, ragged slices included."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for rank, out in res:
        for total, (calls, gp, gre, gim, gc) in out.items():
            assert calls == [shard_range(total, rank, 2)]
            assert gc == [i % 3 + 1 for i in range(total)]
            for i in range(total):
                m = gc[i]
                assert gp[i][:m] == [10 * i + j for j in range(m)]
                assert gre[i][:m] == [float(i)] * m
                assert gim[i][:m] == [-float(j) for j in range(m)]


def test_sharded_batch_without_a_group():
    from paper_2011_05749_b200.shard import sharded_batch

    assert sharded_batch(lambda a, b: (a, b, None), 7) == (0, 7, None)
