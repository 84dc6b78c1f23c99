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
    assert t.is_cuda and t.is_contiguous(), "device tensors must be contiguous CUDA tensors"
    return t.data_ptr()


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
