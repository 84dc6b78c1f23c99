"""Device plumbing: torch owns device memory and streams, the C ABI does the work."""

from __future__ import annotations

import numpy as np
import torch

from . import _lib


def require_cuda():
    if not torch.cuda.is_available():
        raise _lib.FemminCudaError(
            "paper_2109_01158_b200 needs a CUDA device (B200); there is no CPU fallback")
    return _lib.load()


def stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def ptr(t) -> int | None:
    if t is None:
        return None
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.is_contiguous()):
        raise ValueError("device arguments must be contiguous CUDA tensors")
    return t.data_ptr()


def checked(t, name: str, numel: int | None, dtype=torch.float64, *, at_least: bool = False,
            device: int | None = None):
    """Validate a device argument before its raw pointer reaches a kernel:
    a contiguous CUDA tensor of ``dtype`` with ``numel`` elements (or at least
    that many), on ``device``.  Raises ValueError like the reference's shape
    checks (assembly.py:41-46) instead of letting a kernel read or write out of
    bounds.  Returns the tensor (None passes through)."""
    if t is None:
        return None
    if not isinstance(t, torch.Tensor):
        raise ValueError(f"{name} must be a torch CUDA tensor, got {type(t).__name__}")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if device is not None and t.device.index != device:
        raise ValueError(f"{name} is on cuda:{t.device.index}, the context on cuda:{device}")
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if numel is not None:
        n = t.numel()
        if (n < numel) if at_least else (n != numel):
            want = f"at least {numel}" if at_least else f"{numel}"
            raise ValueError(f"{name} has {n} elements, expected {want}")
    return t


def to_dev(a, dtype=None) -> torch.Tensor:
    """Host array (or tensor) -> contiguous CUDA tensor."""
    if isinstance(a, torch.Tensor):
        t = a
    else:
        t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.to("cuda", non_blocking=False).contiguous()


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()
