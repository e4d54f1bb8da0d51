"""Peeling recovery over co-prime cycles (FFAST, R-FFAST) on the GPU.

Drop-in for /root/reference/pkg/src/aliasfft/peeling.py.  Planning
(``plan_cycles`` and its helpers, Kay weights, search-plan shifts and numpy's
seeded anchors) stays on the host: it is integer bookkeeping plus the numpy RNG
draws that parity depends on.  Everything that touches samples or bucket
values runs in the C-ABI library:

* ``build_graph``  → ``afft_build_graph`` (gather + DFT for every cycle/shift),
* ``exact_thresholds`` → ``afft_sumsq`` + ``afft_exact_thresholds``,
* ``classify_exact`` / ``subtract`` → node-batched kernels,
* ``peel_decode`` (exact) → ``afft_peel_exact``: the whole round loop in one
  CTA per signal,
* ``ffast`` → ``afft_ffast``: norm, graph, decode and truncation in one call.

``PeelingGraph`` keeps the reference's host-visible shape (``graph.cycles`` of
``BucketNode`` with ``.state``/``.residual``/``.f0``/``.value``) because callers
inspect nodes after decoding (reference tests/test_peeling.py:250-273); the
throughput path (``batch.ffast_batch``) never materialises nodes on the host.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass, field
from enum import Enum

import numpy as np
import torch

from . import _device, _lib
from .bucketize import SampleLedger, record_bucketization
from .signals import SparseSpectrum


class UnsupportedSizeError(ValueError):
    """A signal size that cannot be split into co-prime cycles (peeling.py:25-26)."""


class NodeState(Enum):
    UNKNOWN = "unknown"
    ZERO_TON = "zero-ton"
    SINGLE_TON = "single-ton"
    MULTI_TON = "multi-ton"
    RESOLVED = "resolved"


# int8 codes shared with include/aliasfft_b200.h (enum afft_node_state)
STATE_CODE = {
    NodeState.UNKNOWN: 0,
    NodeState.ZERO_TON: 1,
    NodeState.SINGLE_TON: 2,
    NodeState.MULTI_TON: 3,
    NodeState.RESOLVED: 4,
}
CODE_STATE = {v: k for k, v in STATE_CODE.items()}


@dataclass
class CyclePlan:
    """Pairwise co-prime bucket counts and the shared shift set (peeling.py:37-46)."""

    factors: list[int]
    shifts: list[int]

    @property
    def r(self) -> int:
        return len(self.shifts)


@dataclass
class SearchPlan:
    """Noisy search layout: c strides 2^j, m rounds each (peeling.py:49-62)."""

    c: int
    m: int
    anchors: list[int]
    weights: np.ndarray
    t0: float | None = None
    t1: float | None = None

    @property
    def shifts(self) -> list[int]:
        return [int(self.anchors[j] + (1 << j) * t) for j in range(self.c) for t in range(self.m)]


class BucketNode:
    """One bucket of one cycle: measurements and live residual (peeling.py:65-75)."""

    def __init__(self, cycle: int, index: int, vec):
        self.cycle = cycle
        self.index = index
        self.vec = np.asarray(vec, dtype=np.complex128)
        self.residual = self.vec.copy()
        self.state = NodeState.UNKNOWN
        self.f0: int | None = None
        self.value: complex | None = None


@dataclass
class PeelingGraph:
    n: int
    factors: list[int]
    shifts: list[int]
    cycles: list[list[BucketNode]]
    recovered: dict[int, complex] = field(default_factory=dict)


@dataclass
class DecodeResult:
    spectrum: SparseSpectrum
    unresolved_multitons: int
    rounds: int
    # extension: check-node identifications of peel_decode(..., decoder="tree")
    identifications: int | None = None


# ------------------------------------------------------------------ planning (host)


def kay_weights(m: int) -> np.ndarray:
    """Parabolic phase-difference weights, summing to 1 (peeling.py:94-99, Eq. 22)."""
    if m < 2:
        raise ValueError("need at least two rounds per iteration")
    t = np.arange(m - 1)
    return 1.5 * m / (m * m - 1.0) * (1.0 - 4.0 * ((2.0 * t - m + 2.0) / (2.0 * m)) ** 2)


def coprime_factors(n: int) -> list[int]:
    """Ascending prime-power factors of n (peeling.py:102-117)."""
    out = []
    rest = n
    p = 2
    while p * p <= rest:
        if rest % p == 0:
            q = 1
            while rest % p == 0:
                rest //= p
                q *= p
            out.append(q)
        p += 1
    if rest > 1:
        out.append(rest)
    return sorted(out)


def _group_factors(powers: list[int], k: int) -> list[int]:
    """Greedy merge into the most cycles that each keep >= 2k buckets (peeling.py:120-134)."""
    target = max(2, 2 * k)
    for d in range(len(powers), 1, -1):
        groups = [1] * d
        for q in sorted(powers, reverse=True):
            groups[groups.index(min(groups))] *= q
        if min(groups) >= target:
            return sorted(groups)
    return list(powers)


def plan_cycles(n: int, k: int, mode: str = "exact", seed: int = 0):
    """Cycle sizes plus shift set; noisy mode adds a seeded SearchPlan (peeling.py:137-166)."""
    powers = coprime_factors(n)
    if len(powers) < 2:
        raise UnsupportedSizeError(
            f"signal size {n} has a single prime-power factor; need two or more co-prime cycles"
        )
    if k**3 >= n:
        warnings.warn(f"peeling works best when k < n^(1/3); got k={k}, n={n}", stacklevel=2)
    factors = _group_factors(powers, k)
    if mode == "exact":
        return CyclePlan(factors=factors, shifts=[0, 1, 2]), None
    if mode != "noisy":
        raise ValueError(f"unknown mode {mode!r}")
    c = int(np.ceil(np.log2(n)))
    m = max(2, int(np.ceil(np.log2(n) ** (1.0 / 3.0))))
    rng = np.random.default_rng(seed)
    anchors = [int(t) for t in rng.integers(0, n, size=c)]
    search = SearchPlan(c=c, m=m, anchors=anchors, weights=kay_weights(m))
    return CyclePlan(factors=factors, shifts=search.shifts), search


# ------------------------------------------------------------------ device graph


def build_graph_device(xd: torch.Tensor, factors, shifts) -> torch.Tensor:
    """(nodes, R) complex128 node measurements for one device signal."""
    n = int(xd.shape[-1])
    factors = [int(b) for b in factors]
    shifts = [int(t) for t in shifts]
    for b in factors:
        if b < 1 or n % b:
            raise ValueError(f"bucket count {b} does not divide signal size {n}")
    total = sum(factors)
    out = torch.empty((total, len(shifts)), dtype=torch.complex128, device=xd.device)
    if total == 0 or not shifts:
        return out
    fb, nc = _lib.host_i64(factors)
    sb, ns = _lib.host_i64(shifts)
    _lib.check(
        _lib.load().afft_build_graph(
            xd.data_ptr(), _device.dtype_code(xd), n, 1, n, fb, nc, sb, ns, out.data_ptr(),
            _device.stream_ptr(),
        ),
        "build_graph",
    )
    return out


def build_graph(x, plan: CyclePlan, ledger: SampleLedger | None = None) -> PeelingGraph:
    """Bucketize every cycle at every shift (peeling.py:169-178) in one launch."""
    n = _device.signal_length(x)
    xd = _device.as_device_signal(x)
    vals = build_graph_device(xd, plan.factors, plan.shifts).cpu().numpy()
    for b in plan.factors:
        record_bucketization(ledger, n, int(b), plan.shifts)
    cycles = []
    g = 0
    for j, b in enumerate(plan.factors):
        cycles.append([BucketNode(j, i, vals[g + i]) for i in range(int(b))])
        g += int(b)
    return PeelingGraph(n=n, factors=list(plan.factors), shifts=list(plan.shifts), cycles=cycles)


def exact_thresholds_device(xd: torch.Tensor) -> torch.Tensor:
    """eps = 1e-6 * ||x|| / sqrt(n) as a 1-element device tensor (peeling.py:316-318)."""
    n = int(xd.shape[-1])
    lib = _lib.load()
    code = _device.dtype_code(xd)
    parts = int(lib.afft_sumsq_parts(n, code))
    partials = torch.empty(parts, dtype=torch.float64, device=xd.device)
    eps = torch.empty(1, dtype=torch.float64, device=xd.device)
    sp = _device.stream_ptr()
    _lib.check(lib.afft_sumsq(xd.data_ptr(), code, n, 1, n, partials.data_ptr(), sp), "sumsq")
    _lib.check(
        lib.afft_exact_thresholds(partials.data_ptr(), parts, n, 1, eps.data_ptr(), sp),
        "exact_thresholds",
    )
    return eps


def exact_thresholds(x) -> float:
    """Scale-aware zero/ratio tolerance for exact classification (peeling.py:316-318)."""
    return float(exact_thresholds_device(_device.as_device_signal(x)).item())


# ------------------------------------------------------------------ per-node API


def _tone_vector(f: int, shifts, n: int) -> np.ndarray:
    """Host helper mirroring peeling.py:181-183 (used only for host-side checks)."""
    prod = (np.asarray(shifts, dtype=np.int64) * int(f)) % n
    return np.exp(-2j * np.pi * prod / n)


def subtract(node: BucketNode, f: int, value: complex, shifts, n: int, b: int) -> None:
    """Remove one tone from a node's residual on the device (peeling.py:186-190)."""
    if f % b != node.index:
        raise ValueError(f"frequency {f} does not belong to bucket {node.index} mod {b}")
    dev = _device.require_cuda()
    shifts = [int(t) for t in shifts]
    res = torch.from_numpy(np.ascontiguousarray(node.residual, dtype=np.complex128)).to(dev)
    fs = torch.tensor([int(f)], dtype=torch.int64, device=dev)
    vs = torch.tensor([complex(value)], dtype=torch.complex128, device=dev)
    sb, ns = _lib.host_i64(shifts)
    _lib.check(
        _lib.load().afft_subtract(
            res.data_ptr(), sb, ns, fs.data_ptr(), vs.data_ptr(), 1, n, _device.stream_ptr()
        ),
        "subtract",
    )
    node.residual = res.cpu().numpy()


def classify_exact(node: BucketNode, eps_zero: float, eps_ratio: float, b: int, n: int,
                   shifts=(0, 1, 2)) -> NodeState:
    """Zero/single/multi from three consecutive shifts (peeling.py:193-215), on the device."""
    if tuple(shifts) != (0, 1, 2):
        raise ValueError("exact classification expects the shift set (0, 1, 2)")
    dev = _device.require_cuda()
    res = torch.from_numpy(np.ascontiguousarray(node.residual[:3], dtype=np.complex128)).to(dev)
    idx = torch.tensor([node.index], dtype=torch.int64, device=dev)
    state = torch.zeros(1, dtype=torch.int8, device=dev)
    f0 = torch.full((1,), -1 if node.f0 is None else int(node.f0), dtype=torch.int64, device=dev)
    val = torch.tensor([0j if node.value is None else complex(node.value)],
                       dtype=torch.complex128, device=dev)
    _lib.check(
        _lib.load().afft_classify_exact(
            res.data_ptr(), idx.data_ptr(), 1, b, n, float(eps_zero), float(eps_ratio),
            state.data_ptr(), f0.data_ptr(), val.data_ptr(), _device.stream_ptr(),
        ),
        "classify_exact",
    )
    node.state = CODE_STATE[int(state.item())]
    if node.state is NodeState.SINGLE_TON:
        node.f0 = int(f0.item())
        node.value = complex(val.item())
    return node.state


# ------------------------------------------------------------------ decoding


def _graph_to_device(graph: PeelingGraph, dev):
    nodes = [node for cyc in graph.cycles for node in cyc]
    r = len(graph.shifts)
    res = np.empty((len(nodes), r), dtype=np.complex128)
    st = np.empty(len(nodes), dtype=np.int8)
    f0 = np.empty(len(nodes), dtype=np.int64)
    val = np.empty(len(nodes), dtype=np.complex128)
    for g, node in enumerate(nodes):
        res[g] = node.residual
        st[g] = STATE_CODE[node.state]
        f0[g] = -1 if node.f0 is None else int(node.f0)
        val[g] = 0j if node.value is None else complex(node.value)
    to = lambda a: torch.from_numpy(a).to(dev)  # noqa: E731
    return nodes, to(res), to(st), to(f0), to(val)


def _graph_from_device(nodes, res, st, f0, val) -> None:
    res, st, f0, val = res.cpu().numpy(), st.cpu().numpy(), f0.cpu().numpy(), val.cpu().numpy()
    for g, node in enumerate(nodes):
        node.residual = res[g].copy()
        node.state = CODE_STATE[int(st[g])]
        if f0[g] >= 0:
            node.f0 = int(f0[g])
            node.value = complex(val[g])


def peel_decode(graph: PeelingGraph, mode: str = "exact", eps_zero: float = 0.0,
                eps_ratio: float = 0.0, search_plan: SearchPlan | None = None,
                max_rounds: int | None = None, *, decoder: str = "rounds") -> DecodeResult:
    """Synchronous peeling (peeling.py:270-313), whole round loop on the device.

    ``decoder="tree"`` (keyword-only, an extension; exact mode) runs the paper's Fig. 5
    tree-walk decoder instead (a non-goal of the reference,
    SPEC.md:460): paths extended from single-ton check nodes, only the d check nodes of
    each decoded tone re-identified (afft_peel_tree_exact).  The recovered set is the
    round decoder's; the insertion order is the walk's; ``rounds`` counts the walk's
    generations and ``identifications`` the check-node identifications."""
    if decoder not in ("rounds", "tree"):
        raise ValueError(f"unknown decoder {decoder!r}")
    if max_rounds is None:
        max_rounds = len(graph.recovered) + 8
    if mode != "exact":
        if decoder == "tree":
            raise ValueError("the tree-walk decoder is exact-mode only")
        return peel_decode_noisy(graph, search_plan, max_rounds)
    live = any(
        node.state not in (NodeState.RESOLVED, NodeState.ZERO_TON)
        for cyc in graph.cycles for node in cyc
    )
    if max_rounds > 0 and live and tuple(graph.shifts) != (0, 1, 2):
        raise ValueError("exact classification expects the shift set (0, 1, 2)")
    dev = _device.require_cuda()
    nodes, res, st, f0, val = _graph_to_device(graph, dev)
    prior = list(graph.recovered.items())
    cap = len(prior) + max(1, len(nodes))
    rec_pos = torch.zeros(cap, dtype=torch.int64)
    rec_val = torch.zeros(cap, dtype=torch.complex128)
    if prior:
        rec_pos[: len(prior)] = torch.tensor([f for f, _ in prior], dtype=torch.int64)
        rec_val[: len(prior)] = torch.tensor([complex(v) for _, v in prior], dtype=torch.complex128)
    rec_pos, rec_val = rec_pos.to(dev), rec_val.to(dev)
    rec_count = torch.tensor([len(prior)], dtype=torch.int32, device=dev)
    eps0 = torch.tensor([float(eps_zero)], dtype=torch.float64, device=dev)
    epsr = torch.tensor([float(eps_ratio)], dtype=torch.float64, device=dev)
    rounds = torch.zeros(1, dtype=torch.int32, device=dev)
    unresolved = torch.zeros(1, dtype=torch.int32, device=dev)
    ident = torch.zeros(1, dtype=torch.int32, device=dev)
    if nodes:
        fb, nc = _lib.host_i64(graph.factors)
        if decoder == "tree":
            _lib.check(
                _lib.load().afft_peel_tree_exact(
                    graph.n, 1, fb, nc, res.data_ptr(), st.data_ptr(), f0.data_ptr(),
                    val.data_ptr(), eps0.data_ptr(), epsr.data_ptr(), rec_pos.data_ptr(),
                    rec_val.data_ptr(), cap, rec_count.data_ptr(), rounds.data_ptr(),
                    unresolved.data_ptr(), ident.data_ptr(), _device.stream_ptr(),
                ),
                "peel_decode",
            )
        else:
            _lib.check(
                _lib.load().afft_peel_exact(
                    graph.n, 1, fb, nc, res.data_ptr(), st.data_ptr(), f0.data_ptr(),
                    val.data_ptr(), eps0.data_ptr(), epsr.data_ptr(), int(max_rounds),
                    rec_pos.data_ptr(), rec_val.data_ptr(), cap, rec_count.data_ptr(),
                    rounds.data_ptr(), unresolved.data_ptr(), _device.stream_ptr(),
                ),
                "peel_decode",
            )
        _graph_from_device(nodes, res, st, f0, val)
    count = int(rec_count.item())
    pos = rec_pos[:count].cpu().numpy()
    vals = rec_val[:count].cpu().numpy()
    for i in range(len(prior), count):
        graph.recovered[int(pos[i])] = complex(vals[i])
    n_rounds = int(rounds.item()) if nodes else max(0, min(1, int(max_rounds)))
    spectrum = SparseSpectrum(graph.n, dict(graph.recovered))
    return DecodeResult(spectrum=spectrum, unresolved_multitons=int(unresolved.item()),
                        rounds=n_rounds,
                        identifications=int(ident.item()) if decoder == "tree" else None)


def ffast(x, k: int, ledger: SampleLedger | None = None, max_rounds: int | None = None, *,
          plan: CyclePlan | None = None) -> SparseSpectrum:
    """Exact peeling decoder, reads 3*(B_1+...+B_d) samples (peeling.py:321-332).

    ``plan`` (keyword-only, an extension) runs an explicit cycle plan, as the
    BASELINE configs need; by default the reference planner chooses it.
    """
    n = _device.signal_length(x)
    if plan is None:
        plan, _ = plan_cycles(n, k, "exact")
    if tuple(plan.shifts) != (0, 1, 2):
        raise ValueError("exact classification expects the shift set (0, 1, 2)")
    from .batch import ffast_batch

    out = ffast_batch(_device.as_device_signal(x).unsqueeze(0), k, plan.factors,
                      max_rounds=max_rounds)
    for b in plan.factors:
        record_bucketization(ledger, n, int(b), plan.shifts)
    if not k:
        return SparseSpectrum(n, {})
    return out.spectrum(0)


from .rffast import (  # noqa: E402  (R-FFAST device paths, re-exported like the reference)
    classify_noisy,
    noisy_thresholds,
    peel_decode_noisy,
    r_ffast,
    robust_thresholds,
    singleton_search_noisy,
)
