"""The signal-sharded harness over the real decoders (C1-C5 are batches of
independent signals): two processes, each decoding its own slice on cuda:0 and exchanging
only the result slots (gloo here — one GPU; NCCL on a multi-GPU node), must end with
exactly the slots of the unsharded call.  No kernel of one rank waits on another rank's."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _inputs():
    from paper_2011_05749_b200 import DsfftConfig, generate_test_case, plan_cycles

    out = {}
    n, k = 124950, 40  # config 1, 5 signals (ragged over 2 ranks)
    out["ffast"] = (np.stack([generate_test_case(n, k, "exact", seed=s).signal for s in range(5)]),
                    k, [49, 50, 51])
    n, k = 4095, 4  # R-FFAST with each signal's own search plan
    plans = [plan_cycles(n, k, "noisy", seed=s) for s in range(5)]
    out["rffast"] = (np.stack([generate_test_case(n, k, 15.0, seed=s).signal for s in range(5)]),
                     k, list(plans[0][0].factors), [p[1] for p in plans])
    n, k = 1 << 16, 64  # sFFT-DT3 with per-signal seeds
    out["dt"] = (np.stack([generate_test_case(n, k, "exact", seed=s).signal for s in range(6)]),
                 k, 256, list(range(6)))
    n, k = 1 << 16, 32  # DSFFT, noisy, per-signal configs
    out["dsfft"] = (np.stack([generate_test_case(n, k, 20.0, seed=s).signal for s in range(3)]),
                    k, [DsfftConfig(mode="noisy", seed=s, noise_std=float(np.sqrt(k * 0.01)))
                        for s in range(3)])
    return out


def _decode_all(group_ready: bool):
    from paper_2011_05749_b200 import shard

    torch.cuda.set_device(0)
    inp = _inputs()
    res = {}
    x, k, f = inp["ffast"]
    res["ffast"] = shard.ffast_sharded(torch.from_numpy(x).cuda(), k, f)
    x, k, f, searches = inp["rffast"]
    res["rffast"] = shard.rffast_sharded(torch.from_numpy(x).cuda(), k, f, searches)
    x, k, b, seeds = inp["dt"]
    res["dt"] = shard.sfft_dt_sharded(torch.from_numpy(x).cuda(), k, b, 4, 12, "dt3", seeds=seeds)
    x, k, cfgs = inp["dsfft"]
    res["dsfft"] = shard.dsfft_sharded(torch.from_numpy(x).cuda(), k, cfgs)
    torch.cuda.synchronize()
    return {name: tuple(t.cpu().numpy() for t in r) for name, r in res.items()}


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, _decode_all(True)))
    finally:
        dist.destroy_process_group()


def test_sharded_decoders_equal_unsharded():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    want = _decode_all(False)  # no process group here: the whole batch on this process
    for rank in (0, 1):
        for name, (wp, wv, wc) in want.items():
            gp, gv, gc = got[rank][name]
            assert np.array_equal(gc, wc), (rank, name)
            assert wc.sum() > 0, name
            for i, m in enumerate(wc):
                assert np.array_equal(gp[i, :m], wp[i, :m]), (rank, name, i)
                assert np.array_equal(gv[i, :m], wv[i, :m]), (rank, name, i)
