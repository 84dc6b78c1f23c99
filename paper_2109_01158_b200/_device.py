"""Device plumbing: torch owns device memory and streams, the C ABI does the work."""

from __future__ import annotations

import os

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


# Large host <-> device transfers of the numpy drop-in go through pinned
# buffers from torch's caching host allocator: a pageable D2H into a fresh
# numpy array page-faults its way through the destination (47 ms for a cfg4
# gradient on the B200 box, tools/copy_probe.py) where a pinned one is a
# 1.9 ms DMA; uploads are copied into pinned memory by host threads (3 ms)
# and DMA'd (1.9 ms) instead of one pageable copy (9 ms).
_PINNED_MIN = 4 << 20  # bytes
_POOL = None


def _copy_threads():
    global _POOL
    if _POOL is None:
        from concurrent.futures import ThreadPoolExecutor
        _POOL = ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 1))
    return _POOL


def _par_copyto(dst: np.ndarray, src: np.ndarray):
    n = dst.shape[0]
    parts = _copy_threads()._max_workers
    cuts = [n * i // parts for i in range(parts + 1)]
    list(_copy_threads().map(lambda i: np.copyto(dst[cuts[i]:cuts[i + 1]],
                                                 src[cuts[i]:cuts[i + 1]]), range(parts)))


def to_dev(a, dtype=None) -> torch.Tensor:
    """Host array (or tensor) -> contiguous CUDA tensor (stream-ordered on the
    current stream)."""
    if isinstance(a, torch.Tensor):
        t = a if dtype is None else a.to(dtype)
        return t.to("cuda", non_blocking=False).contiguous()
    arr = np.ascontiguousarray(a)
    if dtype is not None:
        arr = arr.astype(torch.empty(0, dtype=dtype).numpy().dtype, copy=False)
    if arr.nbytes < _PINNED_MIN or arr.ndim == 0:
        return torch.from_numpy(arr).to("cuda", non_blocking=False).contiguous()
    pin = torch.empty(arr.shape, dtype=torch.from_numpy(arr[:0]).dtype, pin_memory=True)
    out = torch.empty(arr.shape, dtype=pin.dtype, device="cuda")
    # pipelined: the host threads copy consecutive pieces into the pinned
    # buffer while the DMA engine uploads the pieces already copied (the
    # copies take longer than the DMA: cfg4 field 3 + 1.9 ms serial)
    src = arr.reshape(arr.shape[0], -1)
    dst, dev = pin.numpy().reshape(arr.shape[0], -1), out.view(arr.shape[0], -1)
    n, pieces = src.shape[0], 4 * _copy_threads()._max_workers
    cuts = [n * i // pieces for i in range(pieces + 1)]
    futs = [_copy_threads().submit(np.copyto, dst[cuts[i]:cuts[i + 1]], src[cuts[i]:cuts[i + 1]])
            for i in range(pieces)]
    pin_rows = pin.view(arr.shape[0], -1)
    for i, f in enumerate(futs):
        f.result()
        if cuts[i + 1] > cuts[i]:
            # the caching host allocator keeps `pin` until this copy has completed
            dev[cuts[i]:cuts[i + 1]].copy_(pin_rows[cuts[i]:cuts[i + 1]], non_blocking=True)
    return out


def to_host(t: torch.Tensor) -> np.ndarray:
    """CUDA tensor -> numpy.  Large results land in a pinned buffer from
    torch's caching host allocator; the returned array views it (and keeps it
    alive), so no host copy or page faulting is needed."""
    t = t.detach()
    if not t.is_cuda or t.numel() * t.element_size() < _PINNED_MIN:
        return t.cpu().numpy()
    out = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    out.copy_(t, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return out.numpy()
