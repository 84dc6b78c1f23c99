"""Hessian utilities of the reference solver (solver.py:344-398; SURVEY §8f
row 4) on the GPU.

* ``hessian_sparsity(mesh, d)`` — the boolean free-dof Hessian pattern
  (``fm_hessian_pattern``: node pairs of every element sorted and
  de-duplicated, expanded to d x d dof blocks on the free dofs), returned as
  the reference's scipy CSR (same indptr / indices, ascending columns).
* ``greedy_coloring(pattern)`` — a distance-2 colouring with the reference's
  contract (columns sharing a row get distinct colours), computed in parallel
  rounds on the GPU (``fm_color_d2``); the colours themselves may differ from
  the sequential greedy sweep.
* ``colored_fd_hessian(gx, x, pattern, step)`` — the reference algorithm for a
  user gradient callable (one perturbed gradient per colour).
* ``fd_hessian_device(dm, v, model, b, conn, dofs_minim, step)`` — the same
  with everything on the device: the engine's exact-gradient kernel per
  colour, perturbation / scatter / symmetrisation kernels, CSR arrays out.

A free dof's gradient only reads the dofs of its node patch, so with any
distance-2 colouring each scattered difference equals the single-column
difference bit for bit: the Hessian does not depend on the colouring.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from ._device import ptr, require_cuda, stream_ptr


def _dev(a, dtype):
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


def hessian_pattern_device(conn, nn: int, d: int, dofs_minim):
    """CSR (indptr, indices) int64 CUDA tensors of the free-dof pattern."""
    lib = require_cuda()
    conn = _dev(conn, torch.int64)
    dm = _dev(dofs_minim, torch.int64)
    ne, nv = conn.shape
    n = dm.numel()
    indptr = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    nnz = C.c_int64(0)
    _lib.check(lib.fm_hessian_pattern(int(nn), ne, nv, int(d), ptr(conn), n, ptr(dm),
                                      ptr(indptr), None, C.byref(nnz), stream_ptr()),
               "fm_hessian_pattern")
    indices = torch.empty(max(nnz.value, 1), dtype=torch.int64, device="cuda")[:nnz.value]
    _lib.check(lib.fm_hessian_pattern(int(nn), ne, nv, int(d), ptr(conn), n, ptr(dm),
                                      ptr(indptr), ptr(indices), C.byref(nnz), stream_ptr()),
               "fm_hessian_pattern")
    return indptr, indices


def _to_scipy(indptr, indices, n, data=None):
    import scipy.sparse as sp
    ip = indptr.cpu().numpy()
    ix = indices.cpu().numpy()
    vals = np.ones(ix.size, dtype=bool) if data is None else data
    return sp.csr_matrix((vals, ix, ip), shape=(n, n))


def hessian_sparsity(mesh, d: int):
    """solver.py:344-357 (boolean pattern, free dofs only)."""
    indptr, indices = hessian_pattern_device(mesh.elems2nodes, mesh.nn, d, mesh.dofs_minim)
    return _to_scipy(indptr, indices, int(np.asarray(mesh.dofs_minim).size))


def color_device(indptr, indices) -> tuple[torch.Tensor, int]:
    """Distance-2 colours (int32 CUDA tensor) of a symmetric CSR pattern."""
    lib = require_cuda()
    n = indptr.numel() - 1
    colors = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")[:n]
    nc = C.c_int32(0)
    _lib.check(lib.fm_color_d2(n, ptr(indptr), ptr(indices), ptr(colors), C.byref(nc),
                               stream_ptr()), "fm_color_d2")
    return colors, int(nc.value)


def greedy_coloring(pattern) -> np.ndarray:
    """solver.py:360-376 contract: columns sharing a row get distinct colours."""
    P = pattern.tocsr()
    P.sort_indices()
    colors, _ = color_device(_dev(P.indptr, torch.int64), _dev(P.indices, torch.int64))
    return colors.cpu().numpy().astype(np.int64)


def colored_fd_hessian(gx, x, pattern, step=1e-6):
    """solver.py:379-398: explicit sparse Hessian by coloured forward
    differences of a gradient callable ``gx`` (free-dof vector in and out)."""
    import scipy.sparse as sp
    colors = greedy_coloring(pattern)
    P = pattern.tocsr()
    P.sort_indices()
    g0 = np.asarray(gx(x))
    n = x.size
    rows = np.repeat(np.arange(n), np.diff(P.indptr))
    vals = np.zeros(P.indices.size)
    for c in range(int(colors.max()) + 1 if n else 0):
        cols = np.flatnonzero(colors == c)
        xp = x.copy()
        xp[cols] += step
        diff = (np.asarray(gx(xp)) - g0) / step
        sel = colors[P.indices] == c
        vals[sel] = diff[rows[sel]]
    H = sp.csr_matrix((vals, P.indices, P.indptr), shape=(n, n))
    return ((H + H.T) * 0.5).tocsr()


def fd_hessian_device(dm, v, model, b, conn, dofs_minim, step=1e-6, colors=None,
                      pattern=None):
    """colored_fd_hessian on the device around ``dm.exact_gradient``: v is the
    full field (CUDA), the Hessian is over the free dofs (dofs_minim order).
    Returns (indptr, indices, values, ncolors) as CUDA tensors / int."""
    lib = require_cuda()
    indptr, indices = pattern if pattern is not None else hessian_pattern_device(
        conn, dm.nn, dm.d, dofs_minim)
    n = indptr.numel() - 1
    if colors is None:
        colors, nc = color_device(indptr, indices)
    else:
        colors = _dev(colors, torch.int32)
        nc = int(colors.max().item()) + 1 if n else 0
    dmin = _dev(dofs_minim, torch.int64)
    g0 = dm.exact_gradient(v, model, b)
    gp = torch.empty_like(g0)
    vp = torch.empty_like(v)
    vals = torch.zeros(indices.numel(), dtype=torch.float64, device="cuda")
    for c in range(nc):
        vp.copy_(v)
        _lib.check(lib.fm_hess_perturb(n, ptr(dmin), ptr(colors), c, float(step), ptr(vp),
                                       stream_ptr()), "fm_hess_perturb")
        dm.exact_gradient(vp, model, b, g=gp)
        _lib.check(lib.fm_hess_scatter(n, ptr(indptr), ptr(indices), ptr(colors), c, ptr(gp),
                                       ptr(g0), float(step), ptr(vals), stream_ptr()),
                   "fm_hess_scatter")
    out = torch.empty_like(vals)
    _lib.check(lib.fm_hess_symmetrize(n, ptr(indptr), ptr(indices), ptr(vals), ptr(out),
                                      stream_ptr()), "fm_hess_symmetrize")
    dm.check()
    return indptr, indices, out, nc
