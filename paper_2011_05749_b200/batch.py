"""Batched, device-resident entry points — the throughput path.

``ffast_batch`` runs FFAST (peeling.py:321-332) over a (batch, n) block of
signals already resident in HBM with one C-ABI call (``afft_ffast``): the
|x|^2 stream for the exact thresholds, the gather + DFT graph build, the
one-CTA-per-signal peeling decoder and the top-k truncation, all enqueued on
the current stream with no host round-trip.  Results stay on the device as
fixed-size slots ``[batch, k]`` plus counts until the caller asks for them.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _device, _lib
from .signals import SparseSpectrum


@dataclass
class FfastBatchResult:
    n: int
    k: int
    pos: torch.Tensor        # [batch, k] int64, sorted by (-|v|, f)
    val: torch.Tensor        # [batch, k] complex128
    count: torch.Tensor      # [batch] int32 (<= k)
    all_pos: torch.Tensor    # [batch, nodes] int64, pre-truncation, insertion order
    all_val: torch.Tensor    # [batch, nodes] complex128
    all_count: torch.Tensor  # [batch] int32
    rounds: torch.Tensor     # [batch] int32
    unresolved: torch.Tensor  # [batch] int32

    def _host(self):
        if not hasattr(self, "_cache"):
            self._cache = {
                name: getattr(self, name).cpu().numpy()
                for name in ("pos", "val", "count", "all_pos", "all_val", "all_count", "rounds",
                             "unresolved")
            }
        return self._cache

    def spectrum(self, i: int) -> SparseSpectrum:
        """Truncated output of signal i, in the reference's rank order."""
        h = self._host()
        c = int(h["count"][i])
        return SparseSpectrum(
            self.n, {int(f): complex(v) for f, v in zip(h["pos"][i, :c], h["val"][i, :c])}
        )

    def full_spectrum(self, i: int) -> SparseSpectrum:
        """Pre-truncation peel_decode spectrum of signal i (insertion order)."""
        h = self._host()
        c = int(h["all_count"][i])
        return SparseSpectrum(
            self.n, {int(f): complex(v) for f, v in zip(h["all_pos"][i, :c], h["all_val"][i, :c])}
        )


def ffast_workspace_bytes(n: int, dtype_code: int, batch: int, factors) -> int:
    fb, nc = _lib.host_i64(factors)
    return int(_lib.load().afft_ffast_workspace_size(n, dtype_code, batch, fb, nc))


def ffast_batch(x, k: int, factors, max_rounds: int | None = None,
                workspace: torch.Tensor | None = None, out: FfastBatchResult | None = None
                ) -> FfastBatchResult:
    """FFAST over a batch of signals with an explicit cycle plan (shifts 0,1,2)."""
    xd = _device.as_device_batch(x)
    batch, n = int(xd.shape[0]), int(xd.shape[1])
    factors = [int(b) for b in factors]
    nodes = sum(factors)
    dev = xd.device
    code = _device.dtype_code(xd)
    ld = int(xd.stride(0)) if batch > 1 else n
    need = ffast_workspace_bytes(n, code, max(batch, 1), factors)
    if need == 0:
        # planning failed inside the library: surface its message
        _lib.check(_lib.AFFT_EINVAL if any(b < 1 or n % b for b in factors) else
                   _lib.AFFT_EUNSUPPORTED, "ffast")
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=dev)
    if out is None:
        out = FfastBatchResult(
            n=n, k=k,
            pos=torch.empty((batch, k), dtype=torch.int64, device=dev),
            val=torch.empty((batch, k), dtype=torch.complex128, device=dev),
            count=torch.empty(batch, dtype=torch.int32, device=dev),
            all_pos=torch.empty((batch, nodes), dtype=torch.int64, device=dev),
            all_val=torch.empty((batch, nodes), dtype=torch.complex128, device=dev),
            all_count=torch.empty(batch, dtype=torch.int32, device=dev),
            rounds=torch.empty(batch, dtype=torch.int32, device=dev),
            unresolved=torch.empty(batch, dtype=torch.int32, device=dev),
        )
    if batch == 0:
        return out
    fb, nc = _lib.host_i64(factors)
    mr = int(max_rounds) if max_rounds else 0
    _lib.check(
        _lib.load().afft_ffast(
            xd.data_ptr(), code, n, batch, ld, fb, nc, int(k), mr, out.pos.data_ptr(),
            out.val.data_ptr(), out.count.data_ptr(), out.all_pos.data_ptr(),
            out.all_val.data_ptr(), out.all_count.data_ptr(), out.rounds.data_ptr(),
            out.unresolved.data_ptr(), workspace.data_ptr(), int(workspace.numel()),
            _device.stream_ptr(),
        ),
        "ffast",
    )
    return out


def spectra_to_numpy(result: FfastBatchResult) -> list[SparseSpectrum]:
    return [result.spectrum(i) for i in range(int(result.count.shape[0]))]


