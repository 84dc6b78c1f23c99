"""Field layout, element gradients, loads and the total energy (GPU).

Mirror of ``/root/reference/pkg/src/femmin/assembly.py``.  ``energy`` is one
streaming pass of the fused element kernel (csrc/fm_eval_ref.cu ``k_energy``)
over the element records of the cached device context, plus a
fixed-order ``b.v``; loads are assembled on the GPU from the mass-matrix rows.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp
import torch

from . import _lib
from ._device import ptr, require_cuda, stream_ptr, to_dev, to_host
from .device import attach, attached, context_for
from .mesh import Mesh


def flatten(V: np.ndarray) -> np.ndarray:
    """Interleaved flat vector of an (nn, d) coefficient matrix (assembly.py:18-20)."""
    return np.ascontiguousarray(V).ravel()


def unflatten(v: np.ndarray, d: int) -> np.ndarray:
    """assembly.py:23-24."""
    return v.reshape(-1, d)


def gather(V: np.ndarray, connectivity: np.ndarray):
    """Per-component nodal values on element rows (assembly.py:27-32)."""
    Vd = to_dev(np.asarray(V, dtype=np.float64))
    idx = to_dev(np.asarray(connectivity, dtype=np.int64))
    return [to_host(Vd[:, j][idx]) for j in range(Vd.shape[1])]


def evaluate_F(dphi, v_vals):
    """F[j][m] = sum_l v[j][:, l] * dphi[m][:, l] (assembly.py:35-49), GPU, numpy
    einsum summation order."""
    rows = np.asarray(dphi[0]).shape
    for vj in v_vals:
        if np.asarray(vj).shape != rows:
            raise ValueError(f"shape mismatch: values {np.asarray(vj).shape} vs gradients {rows}")
    lib = require_cuda()
    dim, d = len(dphi), len(v_vals)
    nrow = rows[0]
    vals = to_dev(np.stack([np.asarray(vj, dtype=np.float64) for vj in v_vals]))
    dp = to_dev(np.stack([np.asarray(g, dtype=np.float64) for g in dphi]))
    F = torch.empty((d * dim, nrow), dtype=torch.float64, device="cuda")
    _lib.check(lib.fm_eval_F(dim, d, nrow, ptr(vals), ptr(dp), ptr(F), stream_ptr()))
    Fh = to_host(F)
    return [[Fh[j * dim + m] for m in range(dim)] for j in range(d)]


def assemble_mass_matrix(mesh: Mesh) -> sp.csr_matrix:
    """P1 mass matrix from the exact local formula (assembly.py:52-62); the COO
    entries are formed on the GPU, the CSR container is scipy's."""
    nv = mesh.dim + 1
    dev = attached(mesh) or {}
    vol = dev.get("volumes")
    vol = to_dev(np.asarray(mesh.volumes)) if vol is None else vol
    conn = dev.get("conn")
    conn = to_dev(np.asarray(mesh.elems2nodes, dtype=np.int64)) if conn is None else conn
    local = (torch.ones((nv, nv), dtype=torch.float64, device="cuda")
             + torch.eye(nv, dtype=torch.float64, device="cuda")) / (nv * (nv + 1))
    vals = vol[:, None, None] * local[None]
    rows = conn.repeat_interleave(nv, dim=1).reshape(-1)
    cols = conn.repeat(1, nv).reshape(-1)
    M = sp.coo_matrix((to_host(vals).ravel(), (to_host(rows), to_host(cols))),
                      shape=(mesh.nn, mesh.nn))
    return M.tocsr()


@dataclass(frozen=True)
class LinearLoad:
    """Consistent nodal load b[j] = M f[j], flattened to dof order (assembly.py:65-86)."""

    b: np.ndarray

    @classmethod
    def assemble(cls, mesh: Mesh, f, d: int, M: sp.csr_matrix | None = None):
        """Constant d-vector or nodal (nn, d) f; GPU mass-row assembly unless an
        explicit matrix M is supplied."""
        f = np.asarray(f, dtype=float)
        if M is not None:
            F = np.broadcast_to(np.atleast_1d(f), (mesh.nn, d)) if f.ndim <= 1 else f
            return cls(b=flatten(np.column_stack([M @ F[:, j] for j in range(d)])))
        lib = require_cuda()
        dev = attached(mesh) or {}
        vol = dev.get("volumes")
        vol = to_dev(np.asarray(mesh.volumes)) if vol is None else vol
        conn = dev.get("conn")
        conn = to_dev(np.asarray(mesh.elems2nodes, dtype=np.int64)) if conn is None else conn
        b = torch.empty(mesh.nn * d, dtype=torch.float64, device="cuda")
        if f.ndim <= 1:
            fv = np.broadcast_to(np.atleast_1d(f), (d,)).astype(np.float64)
            _lib.check(lib.fm_load_constant(mesh.dim, d, mesh.nn, mesh.ne, ptr(conn), ptr(vol),
                                            (C.c_double * d)(*fv), ptr(b), stream_ptr()))
        else:
            fd = to_dev(np.ascontiguousarray(f.reshape(mesh.nn, d), dtype=np.float64))
            _lib.check(lib.fm_load_nodal(mesh.dim, d, mesh.nn, mesh.ne, ptr(conn), ptr(vol),
                                         ptr(fd), ptr(b), stream_ptr()))
        out = cls(b=to_host(b))
        attach(out, b=b)
        return out

    @classmethod
    def zero(cls, mesh: Mesh, d: int):
        return cls(b=np.zeros(d * mesh.nn))


def _load_device(load):
    if load is None:
        return None
    dev = attached(load)
    if dev and "b" in dev:
        return dev["b"]
    b = to_dev(np.asarray(load.b, dtype=np.float64))
    attach(load, b=b)
    return b


def linear_term(load: LinearLoad, v: np.ndarray) -> float:
    """b . v (assembly.py:89-91), fixed-order device reduction."""
    lib = require_cuda()
    b = _load_device(load)
    vd = to_dev(np.asarray(v, dtype=np.float64))
    if vd.numel() != b.numel():
        raise ValueError(f"field has {vd.numel()} entries, load has {b.numel()}")
    out = torch.empty(3, dtype=torch.float64, device="cuda")
    _lib.check(lib.fm_dot(b.numel(), ptr(b), ptr(vd), ptr(out), stream_ptr()))
    return float(out[0].item())


def _check_field(v, mesh, d):
    v = np.asarray(v, dtype=np.float64)
    if v.ndim != 1 or v.size != d * mesh.nn:
        raise ValueError(f"field has shape {v.shape}, expected ({d * mesh.nn},)")
    return v


def energy(v: np.ndarray, mesh: Mesh, model, load: LinearLoad | None = None):
    """Total energy J(v) plus per-element densities (assembly.py:94-106);
    inadmissible states give J = +inf."""
    d = model.d
    v = _check_field(v, mesh, d)
    ctx = context_for(mesh, None, d)
    vd = to_dev(v)
    dens = torch.empty(mesh.ne, dtype=torch.float64, device="cuda")
    with ctx.lock:
        J = torch.empty(3, dtype=torch.float64, device="cuda")
        ctx.energy(vd, model, _load_device(load), dens, out=J)
        Jh = to_host(J)
        return float(Jh[0]), to_host(dens)


def interpolate(fn, mesh: Mesh, d: int) -> np.ndarray:
    """Flat nodal interpolant of a coordinate function (assembly.py:109-120)."""
    V = np.asarray(fn(mesh.nodes2coord), dtype=float)
    if V.ndim == 1:
        V = V[:, None]
    if V.shape != (mesh.nn, d):
        raise ValueError(f"interpolant has shape {V.shape}, expected {(mesh.nn, d)}")
    return flatten(V)
