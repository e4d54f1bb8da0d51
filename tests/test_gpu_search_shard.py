"""One huge R-FFAST decode split over ranks (SURVEY §8(e) stretch row): the singleton
search's candidate chunks are divided round-robin, partial minima are exchanged once
per peeling round, and the result must equal the single-rank decode bit for bit.

Here the ranks are host threads on one GPU, each on its own stream with its own copy
of all state; the exchange is a host-side barrier + element-wise minimum (no kernel
waits on another).  The NCCL form of the exchange is SearchShard.from_process_group,
covered over gloo in tests/test_shard_gloo.py."""

import threading

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _thread_shards(world):
    barrier = threading.Barrier(world, timeout=120)
    box = [None] * world
    from paper_2011_05749_b200.shard import SearchShard

    def make(rank):
        def reduce_min(scores, cands):
            box[rank] = (scores.cpu().numpy(), cands.cpu().numpy())
            barrier.wait()
            s = np.minimum.reduce([b[0] for b in box])
            c = np.minimum.reduce([b[1] for b in box])
            barrier.wait()  # everyone has read the mailboxes
            scores.copy_(torch.from_numpy(s))
            cands.copy_(torch.from_numpy(c))

        return SearchShard(rank, world, reduce_min)

    return [make(r) for r in range(world)]


@pytest.mark.parametrize("world", [2, 3])
def test_split_search_equals_single_rank(world):
    from paper_2011_05749_b200 import generate_test_case, plan_cycles, rffast_batch

    n, k = 511 * 512 * 513, 1000
    x = torch.from_numpy(np.stack([generate_test_case(n, k, 20.0, seed=s).signal
                                   for s in range(2)])).cuda()
    _, search = plan_cycles(n, k, "noisy", seed=0)
    factors = [511, 512, 513]
    ref = rffast_batch(x, k, factors, search)
    torch.cuda.synchronize()
    shards = _thread_shards(world)
    outs, errors = [None] * world, []

    def run(r):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                outs[r] = rffast_batch(x, k, factors, search, shard=shards[r])
            s.synchronize()
        except Exception as exc:  # noqa: BLE001 - reported below
            errors.append(exc)

    threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for out in outs:  # slots past each signal's count are unwritten: compare the valid ones
        assert torch.equal(out.count, ref.count) and torch.equal(out.all_count, ref.all_count)
        assert torch.equal(out.rounds, ref.rounds)
        for i in range(x.shape[0]):
            c, ac = int(ref.count[i]), int(ref.all_count[i])
            assert torch.equal(out.pos[i, :c], ref.pos[i, :c])
            assert torch.equal(out.val[i, :c], ref.val[i, :c])
            assert torch.equal(out.all_pos[i, :ac], ref.all_pos[i, :ac])
            assert torch.equal(out.all_val[i, :ac], ref.all_val[i, :ac])
