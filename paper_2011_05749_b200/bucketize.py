"""Aliasing-filter encoder on the GPU: shift, subsample, small DFT.

Drop-in for /root/reference/pkg/src/aliasfft/bucketize.py.  ``bucketize`` /
``bucketize_set`` run the gather + DFT kernel (csrc/bucketize.cu) through
``afft_bucketize``; the ``SampleLedger`` is replayed on the host from the
deterministic index formula (j*(n/b) - tau) mod n (bucketize.py:96-98), so the
kernel never has to report which samples it read.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _lib


class SampleLedger:
    """Raw read count plus the set of touched indices (bucketize.py:21-50)."""

    def __init__(self, n: int):
        if n < 1:
            raise ValueError("signal size must be >= 1")
        self.n = n
        self.count = 0
        self._mask = np.zeros(n, dtype=bool)

    def record(self, indices) -> None:
        idx = np.asarray(indices)
        self.count += int(idx.size)
        self._mask[idx] = True

    @property
    def unique_count(self) -> int:
        return int(self._mask.sum())

    @property
    def touched(self) -> set[int]:
        return set(np.flatnonzero(self._mask).tolist())

    @property
    def sampled_fraction(self) -> float:
        return self.unique_count / self.n


@dataclass
class FilteredSpectrum:
    """B bucket values measured at shift tau (bucketize.py:53-63)."""

    b: int
    tau: int
    values: np.ndarray

    def __post_init__(self):
        if len(self.values) != self.b:
            raise ValueError("values length must equal bucket count")


def gather_indices(n: int, b: int, tau: int) -> np.ndarray:
    """The time indices one bucketization reads (bucketize.py:96)."""
    return (np.arange(b, dtype=np.int64) * (n // b) - int(tau)) % n


def record_bucketization(ledger: SampleLedger | None, n: int, b: int, shifts) -> None:
    """Replay ledger.record for each shift: the index set of one bucketization is the
    residue class (-tau) mod L of stride L = n/b, so it is recorded as a strided slice."""
    if ledger is None:
        return
    step = n // b
    for tau in shifts:
        ledger.count += b
        ledger._mask[(-int(tau)) % step::step] = True


def shift(x, tau: int):
    """Rotated signal x'[i] = x[(i - tau) mod N] (bucketize.py:66-68); index helper."""
    if isinstance(x, torch.Tensor):
        return torch.roll(x, int(tau))
    return np.roll(np.asarray(x), tau)


def downsample(x, step: int, ledger: SampleLedger | None = None):
    """x[0], x[step], ... ; step must divide len(x) (bucketize.py:71-80); index helper."""
    size = _device.signal_length(x) if isinstance(x, torch.Tensor) else np.asarray(x).size
    if step < 1 or size % step:
        raise ValueError(f"subsampling step {step} does not divide signal size {size}")
    if ledger is not None:
        ledger.record(np.arange(0, size, step))
    if isinstance(x, torch.Tensor):
        return x[::step]
    return np.asarray(x)[::step]


def _check_divides(n: int, b: int) -> None:
    if b < 1 or n % b:
        raise ValueError(f"bucket count {b} does not divide signal size {n}")


def bucketize_device(xd: torch.Tensor, b: int, shifts) -> torch.Tensor:
    """Device core: (len(shifts), b) complex128 tensor of bucket values."""
    n = int(xd.shape[-1])
    _check_divides(n, b)
    shifts = [int(t) for t in shifts]
    out = torch.empty((len(shifts), b), dtype=torch.complex128, device=xd.device)
    if not shifts:
        return out
    buf, cnt = _lib.host_i64(shifts)
    lib = _lib.load()
    _lib.check(
        lib.afft_bucketize(
            xd.data_ptr(), _device.dtype_code(xd), n, 1, n, b, buf, cnt, out.data_ptr(),
            len(shifts) * b, b, 1, _device.stream_ptr(),
        ),
        "bucketize",
    )
    return out


def bucketize(x, b: int, tau: int, ledger: SampleLedger | None = None) -> FilteredSpectrum:
    """Shift by tau, subsample to b points, size-b DFT / b (bucketize.py:83-99)."""
    n = _device.signal_length(x)
    _check_divides(n, b)
    xd = _device.as_device_signal(x)
    vals = bucketize_device(xd, b, [tau])[0]
    record_bucketization(ledger, n, b, [tau])
    return FilteredSpectrum(b=b, tau=tau, values=vals.cpu().numpy())


def bucketize_set(x, b: int, shifts, ledger: SampleLedger | None = None) -> list[FilteredSpectrum]:
    """One FilteredSpectrum per shift, in order, from a single launch (bucketize.py:102-106)."""
    n = _device.signal_length(x)
    _check_divides(n, b)
    shifts = [int(t) for t in shifts]
    xd = _device.as_device_signal(x)
    vals = bucketize_device(xd, b, shifts).cpu().numpy()
    record_bucketization(ledger, n, b, shifts)
    return [FilteredSpectrum(b=b, tau=t, values=vals[i].copy()) for i, t in enumerate(shifts)]
