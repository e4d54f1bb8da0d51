"""Device plumbing: signals as CUDA tensors, the current stream, workspaces.

PyTorch is used only for device memory and streams; all arithmetic on the hot
path runs in the C-ABI library.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib


class NoCudaDevice(RuntimeError):
    """Raised when the hot path is called without a CUDA device (no CPU fallback)."""


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise NoCudaDevice(
            "paper_2011_05749_b200 runs its hot path on a CUDA (B200, sm_100a) device only; "
            "no CUDA device is visible and there is no CPU fallback"
        )
    _lib.load()
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.complex64:
        return _lib.AFFT_C64
    if t.dtype == torch.complex128:
        return _lib.AFFT_C128
    raise ValueError(f"signal dtype {t.dtype} is not complex64/complex128")


def as_device_signal(x) -> torch.Tensor:
    """1-D complex signal on the current CUDA device.

    complex64 stays complex64 (its upcast to complex128, which the reference
    does at bucketize.py:91, is exact and happens in-register at the gather);
    every other dtype becomes complex128 like ``np.asarray(x, complex128)``.
    """
    dev = require_cuda()
    if isinstance(x, torch.Tensor):
        t = x
        if t.dtype not in (torch.complex64, torch.complex128):
            t = t.to(torch.complex128)
        t = t.to(dev)
    else:
        a = np.asarray(x)
        if a.dtype != np.complex64:
            a = np.asarray(a, dtype=np.complex128)
        t = torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    if t.dim() != 1:
        t = t.reshape(-1)
    return t.contiguous()


def as_device_batch(x) -> torch.Tensor:
    """2-D (batch, n) complex signals on the current CUDA device (rows contiguous)."""
    dev = require_cuda()
    if isinstance(x, torch.Tensor):
        t = x
        if t.dtype not in (torch.complex64, torch.complex128):
            t = t.to(torch.complex128)
        t = t.to(dev)
    else:
        a = np.asarray(x)
        if a.dtype != np.complex64:
            a = np.asarray(a, dtype=np.complex128)
        t = torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    if t.dim() == 1:
        t = t.unsqueeze(0)
    if t.dim() != 2:
        raise ValueError("expected a (batch, n) array of signals")
    if t.stride(1) != 1:
        t = t.contiguous()
    return t


def signal_length(x) -> int:
    if isinstance(x, torch.Tensor):
        return int(x.shape[-1]) if x.dim() else 1
    return len(x)


def c128_view(t: torch.Tensor) -> torch.Tensor:
    """Real (..., 2) float64 view of a complex128 tensor (for numpy-free copies)."""
    return torch.view_as_real(t)


def empty(shape, dtype, device=None) -> torch.Tensor:
    return torch.empty(shape, dtype=dtype, device=device or require_cuda())


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()
