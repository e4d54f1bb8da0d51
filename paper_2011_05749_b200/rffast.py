"""R-FFAST on the GPU: noisy thresholds, exhaustive singleton search, noisy peeling.

Device paths for /root/reference/pkg/src/aliasfft/peeling.py:218-267 and
335-386 (re-exported from ``peeling``).  The search plan (c strides of m rounds,
numpy-seeded anchors, Kay weights) is built on the host by ``plan_cycles``; the
thresholds, the L x c candidate scan, the least-squares fit and every peeling
round run in csrc/rffast.cu.
"""

from __future__ import annotations

import ctypes

from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _lib
from .bucketize import SampleLedger, record_bucketization
from .signals import SparseSpectrum


def _search_args(search):
    shifts = search.shifts
    sb, ns = _lib.host_i64(shifts)
    wb = _lib.host_f64(np.asarray(search.weights, dtype=np.float64).tolist())
    return sb, ns, wb


def _node_workspace(n, count, b, c, m, dev):
    need = int(_lib.load().afft_singleton_workspace_size(n, count, b, c, m))
    if need == 0:
        _lib.check(_lib.AFFT_EUNSUPPORTED, "noisy search plan")
    return torch.empty(need, dtype=torch.uint8, device=dev)


def _workspace(n, batch, factors, c, m, dev):
    fb, nc = _lib.host_i64(factors)
    need = int(_lib.load().afft_noisy_workspace_size(n, batch, fb, nc, c, m))
    if need == 0:
        _lib.check(_lib.AFFT_EUNSUPPORTED, "noisy plan")
    return torch.empty(need, dtype=torch.uint8, device=dev)


def _node_tensors(node, dev):
    res = torch.from_numpy(np.ascontiguousarray(node.residual, dtype=np.complex128)).to(dev)
    idx = torch.tensor([int(node.index)], dtype=torch.int64, device=dev)
    return res, idx


def singleton_search_noisy(node, plan, b: int, n: int):
    """Locate and fit the dominant tone of a bucket under noise (peeling.py:222-250)."""
    c, m = plan.c, plan.m
    if node.residual.size != c * m:
        raise ValueError("node does not carry a full search measurement set")
    dev = _device.require_cuda()
    res, idx = _node_tensors(node, dev)
    f0 = torch.empty(1, dtype=torch.int64, device=dev)
    val = torch.empty(1, dtype=torch.complex128, device=dev)
    rn = torch.empty(1, dtype=torch.float64, device=dev)
    ws = _node_workspace(n, 1, b, c, m, dev)
    sb, ns, wb = _search_args(plan)
    _lib.check(
        _lib.load().afft_singleton_search_noisy(
            res.data_ptr(), idx.data_ptr(), 1, b, n, sb, ns, c, m, wb, f0.data_ptr(),
            val.data_ptr(), rn.data_ptr(), ws.data_ptr(), ws.numel(), _device.stream_ptr(),
        ),
        "singleton_search_noisy",
    )
    return int(f0.item()), complex(val.item()), float(rn.item())


def classify_noisy(node, plan, b: int, n: int):
    """Threshold-based zero/single/multi decision (peeling.py:253-267), on the device."""
    from .peeling import CODE_STATE, NodeState

    if plan.t0 is None or plan.t1 is None:
        raise ValueError("search plan thresholds are not set")
    c, m = plan.c, plan.m
    if node.residual.size != c * m:
        raise ValueError("node does not carry a full search measurement set")
    dev = _device.require_cuda()
    res, idx = _node_tensors(node, dev)
    st = torch.empty(1, dtype=torch.int8, device=dev)
    f0 = torch.empty(1, dtype=torch.int64, device=dev)
    val = torch.empty(1, dtype=torch.complex128, device=dev)
    rn = torch.empty(1, dtype=torch.float64, device=dev)
    ws = _node_workspace(n, 1, b, c, m, dev)
    sb, ns, wb = _search_args(plan)
    _lib.check(
        _lib.load().afft_classify_noisy(
            res.data_ptr(), idx.data_ptr(), 1, b, n, sb, ns, c, m, wb, float(plan.t0),
            float(plan.t1), st.data_ptr(), f0.data_ptr(), val.data_ptr(), rn.data_ptr(),
            ws.data_ptr(), ws.numel(), _device.stream_ptr(),
        ),
        "classify_noisy",
    )
    node.state = CODE_STATE[int(st.item())]
    if node.state is NodeState.SINGLE_TON:
        node.f0 = int(f0.item())
        node.value = complex(val.item())
    return node.state


def robust_thresholds_device(energies: torch.Tensor, r: int, mask: torch.Tensor | None = None):
    """(t0, t1) device tensors [batch] from energies [batch, count] (peeling.py:335-351)."""
    if energies.dim() == 1:
        energies = energies.unsqueeze(0)
    energies = energies.to(torch.float64).contiguous()
    batch, count = energies.shape
    dev = energies.device
    t0 = torch.empty(batch, dtype=torch.float64, device=dev)
    t1 = torch.empty(batch, dtype=torch.float64, device=dev)
    mk = None if mask is None else mask.to(torch.uint8).reshape(batch, count).contiguous()
    _lib.check(
        _lib.load().afft_robust_thresholds(
            energies.data_ptr(), None if mk is None else mk.data_ptr(), count, batch, int(r),
            t0.data_ptr(), t1.data_ptr(), _device.stream_ptr(),
        ),
        "robust_thresholds",
    )
    return t0, t1


def robust_thresholds(energies, r: int, scale=None) -> tuple[float, float]:
    """Zero-ton gate T0 and singleton gate T1 from bucket energies (peeling.py:335-351).

    ``scale`` (the floor's reference, default the energies themselves) is honoured
    by passing the median set as a mask over the concatenation [energies, scale].
    """
    dev = _device.require_cuda()
    e = np.asarray(energies, dtype=np.float64).reshape(-1)
    if scale is None:
        t0, t1 = robust_thresholds_device(torch.from_numpy(e).to(dev), r)
    else:
        s = np.asarray(scale, dtype=np.float64).reshape(-1)
        allv = np.concatenate([e, s])
        mask = np.concatenate([np.ones(e.size, np.uint8), np.zeros(s.size, np.uint8)])
        t0, t1 = robust_thresholds_device(torch.from_numpy(allv).to(dev), r,
                                          torch.from_numpy(mask).to(dev))
    return float(t0.item()), float(t1.item())


def node_energies_device(nodes: torch.Tensor) -> torch.Tensor:
    """||vec||^2 per node of a [..., R] complex128 tensor (peeling.py:355-357)."""
    R = int(nodes.shape[-1])
    count = nodes.numel() // R
    out = torch.empty(nodes.shape[:-1], dtype=torch.float64, device=nodes.device)
    _lib.check(
        _lib.load().afft_node_energies(nodes.data_ptr(), R, count, out.data_ptr(),
                                       _device.stream_ptr()),
        "node_energies",
    )
    return out


def noisy_thresholds(graph) -> tuple[float, float]:
    """T0/T1 from the median node energy of the whole graph (peeling.py:354-358)."""
    dev = _device.require_cuda()
    vec = np.stack([node.vec for cyc in graph.cycles for node in cyc])
    e = node_energies_device(torch.from_numpy(np.ascontiguousarray(vec)).to(dev))
    t0, t1 = robust_thresholds_device(e.reshape(1, -1), len(graph.shifts))
    return float(t0.item()), float(t1.item())


@dataclass
class NoisyDecode:
    rec_pos: torch.Tensor
    rec_val: torch.Tensor
    rec_count: torch.Tensor
    rounds: torch.Tensor
    unresolved: torch.Tensor


def _shard_struct(shard, ws: torch.Tensor):
    """AfftSearchShard whose exchange callback runs shard.reduce_min on views of the
    workspace tensor (the partial arrays live inside it)."""
    if shard is None or shard.world == 1:
        return None, None
    base = ws.data_ptr()
    errors = []

    def exchange(ctx, ps, pt, count, stream):
        try:
            scores = ws[ps - base: ps - base + 8 * count].view(torch.float64)
            cands = ws[pt - base: pt - base + 4 * count].view(torch.int32)
            shard.reduce_min(scores, cands)
            return 0
        except Exception as exc:  # noqa: BLE001 - reported to the C caller as a status
            errors.append(exc)
            return 1

    cb = _lib.EXCHANGE_FN(exchange)
    st = _lib.SearchShardC(shard.rank, shard.world, cb, None)
    return st, (cb, errors)


def peel_noisy_device(n, factors, search, residual, state, node_f0, node_val, t0, t1,
                      max_rounds, rec_pos, rec_val, rec_count, shard=None) -> NoisyDecode:
    """afft_peel_noisy on device tensors shaped [batch, nodes, R] / [batch, nodes];
    with a shard.SearchShard the singleton search is split over its ranks."""
    batch = int(residual.shape[0])
    dev = residual.device
    fb, nc = _lib.host_i64(factors)
    sb, ns, wb = _search_args(search)
    ws = _workspace(n, batch, factors, search.c, search.m, dev)
    rounds = torch.zeros(batch, dtype=torch.int32, device=dev)
    unresolved = torch.zeros(batch, dtype=torch.int32, device=dev)
    sh, keep = _shard_struct(shard, ws)
    rc = _lib.load().afft_peel_noisy_sharded(
        n, batch, fb, nc, sb, ns, search.c, search.m, wb, residual.data_ptr(),
        state.data_ptr(), node_f0.data_ptr(), node_val.data_ptr(), t0.data_ptr(),
        t1.data_ptr(), int(max_rounds), rec_pos.data_ptr(), rec_val.data_ptr(),
        int(rec_pos.shape[-1]), rec_count.data_ptr(), rounds.data_ptr(),
        unresolved.data_ptr(), ws.data_ptr(), ws.numel(), _device.stream_ptr(),
        ctypes.byref(sh) if sh is not None else None,
    )
    if keep is not None and keep[1]:
        raise RuntimeError(f"search shard exchange failed: {keep[1][0]!r}") from keep[1][0]
    _lib.check(rc, "peel_decode(noisy)")
    return NoisyDecode(rec_pos, rec_val, rec_count, rounds, unresolved)


def peel_decode_noisy(graph, search, max_rounds: int):
    """Graph-API noisy peel_decode (peeling.py:270-313), state copied back to the nodes."""
    from .peeling import DecodeResult, _graph_from_device, _graph_to_device

    if search is None or search.t0 is None or search.t1 is None:
        live = any(nd.state.value not in ("resolved", "zero-ton")
                   for cyc in graph.cycles for nd in cyc)
        if live and max_rounds > 0:
            raise ValueError("search plan thresholds are not set")
    dev = _device.require_cuda()
    nodes, res, st, f0, val = _graph_to_device(graph, dev)
    if nodes and res.shape[1] != search.c * search.m:
        raise ValueError("node does not carry a full search measurement set")
    prior = list(graph.recovered.items())
    cap = len(prior) + max(1, len(nodes))
    rec_pos = torch.zeros((1, cap), dtype=torch.int64)
    rec_val = torch.zeros((1, cap), dtype=torch.complex128)
    if prior:
        rec_pos[0, : len(prior)] = torch.tensor([f for f, _ in prior], dtype=torch.int64)
        rec_val[0, : len(prior)] = torch.tensor([complex(v) for _, v in prior],
                                                dtype=torch.complex128)
    rec_pos, rec_val = rec_pos.to(dev), rec_val.to(dev)
    rec_count = torch.tensor([len(prior)], dtype=torch.int32, device=dev)
    n_rounds, unresolved = 0, 0
    if nodes:
        t0 = torch.tensor([float(search.t0 or 0.0)], dtype=torch.float64, device=dev)
        t1 = torch.tensor([float(search.t1 or 0.0)], dtype=torch.float64, device=dev)
        out = peel_noisy_device(graph.n, graph.factors, search, res.unsqueeze(0),
                                st.unsqueeze(0), f0.unsqueeze(0), val.unsqueeze(0), t0, t1,
                                max_rounds, rec_pos, rec_val, rec_count)
        _graph_from_device(nodes, res, st, f0, val)
        n_rounds, unresolved = int(out.rounds.item()), int(out.unresolved.item())
    else:
        n_rounds = max(0, min(1, int(max_rounds)))
    count = int(rec_count.item())
    pos = rec_pos[0, :count].cpu().numpy()
    vals = rec_val[0, :count].cpu().numpy()
    for i in range(len(prior), count):
        graph.recovered[int(pos[i])] = complex(vals[i])
    return DecodeResult(spectrum=SparseSpectrum(graph.n, dict(graph.recovered)),
                        unresolved_multitons=unresolved, rounds=n_rounds)


@dataclass
class RffastBatchResult:
    n: int
    k: int
    pos: torch.Tensor
    val: torch.Tensor
    count: torch.Tensor
    all_pos: torch.Tensor
    all_val: torch.Tensor
    all_count: torch.Tensor
    rounds: torch.Tensor
    unresolved: torch.Tensor
    t0: torch.Tensor
    t1: torch.Tensor

    def spectrum(self, i: int) -> SparseSpectrum:
        c = int(self.count[i])
        pos = self.pos[i, :c].cpu().numpy()
        val = self.val[i, :c].cpu().numpy()
        return SparseSpectrum(self.n, {int(f): complex(v) for f, v in zip(pos, val)})

    def full_spectrum(self, i: int) -> SparseSpectrum:
        c = int(self.all_count[i])
        pos = self.all_pos[i, :c].cpu().numpy()
        val = self.all_val[i, :c].cpu().numpy()
        return SparseSpectrum(self.n, {int(f): complex(v) for f, v in zip(pos, val)})


def rffast_batch(x, k: int, factors, search, max_rounds: int | None = None, *,
                 shard=None) -> RffastBatchResult:
    """R-FFAST over a (batch, n) block: graph build at the c*m search shifts,
    median-energy thresholds, noisy peeling and top-k truncation, all on the device.

    ``search`` is one SearchPlan for every signal or a list with one per signal (the
    reference draws each signal's anchors from its own seed, peeling.py:163-164).
    Unsharded, the whole decode is one stream-ordered afft_rffast enqueue (the
    peeling rounds run as a device-side graph loop).  ``shard`` (a shard.SearchShard)
    splits the singleton search of this same batch over several ranks (one huge
    signal on several GPUs; one shared plan); results are unchanged."""
    xd = _device.as_device_batch(x)
    batch, n = int(xd.shape[0]), int(xd.shape[1])
    dev = xd.device
    factors = [int(b) for b in factors]
    plans = list(search) if isinstance(search, (list, tuple)) else [search] * max(batch, 1)
    if len(plans) != max(batch, 1):
        raise ValueError(f"{len(plans)} search plans for {batch} signals")
    c, m = plans[0].c, plans[0].m
    if any(p.c != c or p.m != m for p in plans):
        raise ValueError("every signal's search plan must share c and m")
    for b in factors:
        if b < 1 or n % b:
            raise ValueError(f"bucket count {b} does not divide signal size {n}")
    if shard is not None and shard.world > 1:
        if any(list(p.anchors) != list(plans[0].anchors) for p in plans):
            raise ValueError("a sharded search needs one search plan for the batch")
        return _rffast_batch_sharded(xd, k, factors, plans[0], max_rounds, shard)
    N = sum(factors)
    kk = max(int(k), 0)
    lib = _lib.load()
    fb, nc = _lib.host_i64(factors)
    need = int(lib.afft_rffast_workspace_size(n, batch, fb, nc, c, m))
    if need == 0:
        _lib.check(_lib.AFFT_EUNSUPPORTED, "r_ffast plan")
    ws = torch.empty(need, dtype=torch.uint8, device=dev)
    same = all(p is plans[0] for p in plans)
    anchors = np.asarray([list(p.anchors) for p in (plans[:1] if same else plans)],
                         dtype=np.int64)
    if anchors.shape[1] != c:
        raise ValueError("search plan anchors must number c")
    ab = anchors.ctypes.data_as(ctypes.c_void_p)
    wb = _lib.host_f64(np.asarray(plans[0].weights, dtype=np.float64).tolist())
    out = RffastBatchResult(
        n, k,
        pos=torch.empty((batch, kk), dtype=torch.int64, device=dev),
        val=torch.empty((batch, kk), dtype=torch.complex128, device=dev),
        count=torch.empty(batch, dtype=torch.int32, device=dev),
        all_pos=torch.empty((batch, N), dtype=torch.int64, device=dev),
        all_val=torch.empty((batch, N), dtype=torch.complex128, device=dev),
        all_count=torch.empty(batch, dtype=torch.int32, device=dev),
        rounds=torch.empty(batch, dtype=torch.int32, device=dev),
        unresolved=torch.empty(batch, dtype=torch.int32, device=dev),
        t0=torch.empty(batch, dtype=torch.float64, device=dev),
        t1=torch.empty(batch, dtype=torch.float64, device=dev),
    )
    if batch == 0:
        return out
    ld = int(xd.stride(0)) if batch > 1 else n
    mr = int(max_rounds) if max_rounds else kk + 4
    _lib.check(lib.afft_rffast(
        xd.data_ptr(), _device.dtype_code(xd), n, batch, ld, fb, nc, ab, 0 if same else c, c, m,
        wb, kk, mr, out.pos.data_ptr(), out.val.data_ptr(), out.count.data_ptr(),
        out.all_pos.data_ptr(), out.all_val.data_ptr(), out.all_count.data_ptr(),
        out.rounds.data_ptr(), out.unresolved.data_ptr(), out.t0.data_ptr(), out.t1.data_ptr(),
        ws.data_ptr(), ws.numel(), _device.stream_ptr()), "r_ffast")
    return out


def _rffast_batch_sharded(xd, k, factors, search, max_rounds, shard) -> RffastBatchResult:
    """The sequence with a split singleton search: graph build, thresholds, then
    afft_peel_noisy_sharded (one partial exchange per round through the shard)."""
    batch, n = int(xd.shape[0]), int(xd.shape[1])
    dev = xd.device
    shifts = search.shifts
    R = len(shifts)
    N = sum(factors)
    nodes = torch.empty((batch, N, R), dtype=torch.complex128, device=dev)
    fb, nc = _lib.host_i64(factors)
    sb, ns = _lib.host_i64(shifts)
    ld = int(xd.stride(0)) if batch > 1 else n
    lib = _lib.load()
    _lib.check(lib.afft_build_graph(xd.data_ptr(), _device.dtype_code(xd), n, batch, ld, fb, nc,
                                    sb, ns, nodes.data_ptr(), _device.stream_ptr()), "build_graph")
    t0, t1 = robust_thresholds_device(node_energies_device(nodes), R)
    state = torch.zeros((batch, N), dtype=torch.int8, device=dev)
    f0 = torch.full((batch, N), -1, dtype=torch.int64, device=dev)
    val = torch.zeros((batch, N), dtype=torch.complex128, device=dev)
    rec_pos = torch.empty((batch, N), dtype=torch.int64, device=dev)
    rec_val = torch.empty((batch, N), dtype=torch.complex128, device=dev)
    rec_count = torch.zeros(batch, dtype=torch.int32, device=dev)
    mr = int(max_rounds) if max_rounds else k + 4
    out = peel_noisy_device(n, factors, search, nodes, state, f0, val, t0, t1, mr, rec_pos,
                            rec_val, rec_count, shard=shard)
    kk = max(int(k), 0)
    opos = torch.empty((batch, kk), dtype=torch.int64, device=dev)
    oval = torch.empty((batch, kk), dtype=torch.complex128, device=dev)
    ocount = torch.empty(batch, dtype=torch.int32, device=dev)
    _lib.check(lib.afft_truncate(rec_pos.data_ptr(), rec_val.data_ptr(), rec_count.data_ptr(), N,
                                 batch, kk, opos.data_ptr(), oval.data_ptr(), ocount.data_ptr(),
                                 _device.stream_ptr()), "truncate")
    return RffastBatchResult(n, k, opos, oval, ocount, rec_pos, rec_val, rec_count, out.rounds,
                             out.unresolved, t0, t1)


def r_ffast(x, k: int, ledger: SampleLedger | None = None, seed: int = 0,
            snr_hint: float | None = None, max_rounds: int | None = None, *, plan=None,
            search=None) -> SparseSpectrum:
    """Noise-robust peeling decoder (peeling.py:361-386); reads c*m*(B_1+...+B_d) samples.

    Keyword-only ``plan``/``search`` (an extension) run an explicit cycle plan
    and search plan, as BASELINE config 3 needs (factors 511/512/513).
    """
    from .peeling import CyclePlan, SearchPlan, kay_weights, plan_cycles

    n = _device.signal_length(x)
    if plan is None or search is None:
        auto_plan, auto_search = plan_cycles(n, k, "noisy", seed)
        plan = plan or auto_plan
        search = search or auto_search
    if snr_hint is not None and snr_hint < 5.0:
        search = SearchPlan(c=search.c, m=search.m + 1, anchors=search.anchors,
                            weights=kay_weights(search.m + 1))
        plan = CyclePlan(factors=plan.factors, shifts=search.shifts)
    if list(plan.shifts) != list(search.shifts):
        raise ValueError("cycle plan shifts must be the search plan's shifts")
    res = rffast_batch(_device.as_device_signal(x).unsqueeze(0), k, plan.factors, search,
                       max_rounds=max_rounds)
    search.t0, search.t1 = float(res.t0[0]), float(res.t1[0])
    for b in plan.factors:
        record_bucketization(ledger, n, int(b), plan.shifts)
    if not k:
        return SparseSpectrum(n, {})
    return res.spectrum(0)
