"""Flat, prefix-indexed nodal patches (GPU): mirror of patches.py (reference).

``build_patches`` runs a stable radix sort of (free-node rank, element) pairs
on the GPU (csrc/fm_prep.cu); lengths, prefix, elems and the owner slots are
bit-exact with the reference's lexsort (patches.py:37-71).  The per-row copies
(volumes, elems2nodes, dphi, logical) are gathered on the device as well.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._device import ptr, require_cuda, stream_ptr, to_dev, to_host
from .device import attach, attached
from .mesh import Mesh, MeshError


class PatchStructureError(MeshError):
    """A free node without adjacent elements was found (patches.py:18-19)."""


@dataclass(frozen=True)
class Patches:
    """patches.py:22-34 (plus ``slot`` = argmax of ``logical``)."""

    lengths: np.ndarray
    elems: np.ndarray
    volumes: np.ndarray
    elems2nodes: np.ndarray
    dphi: list
    logical: np.ndarray
    prefix: np.ndarray
    slot: np.ndarray | None = None

    @property
    def total_rows(self) -> int:
        return self.elems.shape[0]


def build_patches_device(conn_d: torch.Tensor, nodes_minim_d: torch.Tensor, nn: int, nv: int):
    """CSR (prefix, elems, slot) as CUDA tensors; raises PatchStructureError."""
    lib = require_cuda()
    ne = conn_d.shape[0]
    nfree = nodes_minim_d.shape[0]
    lengths = torch.empty(nfree, dtype=torch.int64, device="cuda")
    prefix = torch.empty(nfree, dtype=torch.int64, device="cuda")
    elems = torch.empty(ne * nv, dtype=torch.int64, device="cuda")
    slot = torch.empty(ne * nv, dtype=torch.int64, device="cuda")
    total, bad = C.c_int64(0), C.c_int64(-1)
    _lib.check(lib.fm_build_patches(nn, ne, nv, ptr(conn_d), ptr(nodes_minim_d), nfree,
                                    ptr(lengths), ptr(prefix), ptr(elems), ptr(slot),
                                    C.byref(total), C.byref(bad), stream_ptr()))
    T = total.value
    return prefix, elems[:T], slot[:T]


def build_patches(mesh: Mesh) -> Patches:
    """patches.py:37-71: rows of patch i contiguous, ascending element index."""
    dev = attached(mesh) or {}
    conn_d = dev.get("conn")
    if conn_d is None:
        conn_d = to_dev(np.asarray(mesh.elems2nodes, dtype=np.int64))
    nm_d = dev.get("nodes_minim")
    if nm_d is None:
        nm_d = to_dev(np.asarray(mesh.nodes_minim, dtype=np.int64))
    nv = mesh.elems2nodes.shape[1]
    prefix_d, elems_d, slot_d = build_patches_device(conn_d, nm_d, mesh.nn, nv)
    lengths_d = torch.diff(prefix_d, prepend=torch.zeros(1, dtype=torch.int64, device="cuda"))
    rows_conn = conn_d.index_select(0, elems_d)
    vol_d = dev.get("volumes")
    vol_d = to_dev(np.asarray(mesh.volumes)) if vol_d is None else vol_d
    dphi_d = dev.get("dphi")
    if dphi_d is None:
        dphi_d = to_dev(np.stack([np.asarray(g) for g in mesh.dphi]))
    logical = torch.zeros_like(rows_conn, dtype=torch.bool)
    logical.scatter_(1, slot_d.view(-1, 1), True)
    out = Patches(lengths=to_host(lengths_d), elems=to_host(elems_d),
                  volumes=to_host(vol_d.index_select(0, elems_d)),
                  elems2nodes=to_host(rows_conn),
                  dphi=[to_host(dphi_d[m].index_select(0, elems_d)) for m in range(mesh.dim)],
                  logical=to_host(logical), prefix=to_host(prefix_d), slot=to_host(slot_d))
    attach(out, prefix=prefix_d, elems=elems_d, slot=slot_d)
    return out


def patch_prefix_indices(patches: Patches, d: int) -> np.ndarray:
    """patches.py:74-77: block b shifted by b * ||T||."""
    total = patches.total_rows
    return np.concatenate([np.asarray(patches.prefix) + b * total for b in range(d)])


def segment_sums(values: np.ndarray, indx: np.ndarray) -> np.ndarray:
    """patches.py:80-83 as direct fixed-order per-segment sums on the GPU."""
    lib = require_cuda()
    vals = to_dev(np.asarray(values, dtype=np.float64))
    ind = to_dev(np.asarray(indx, dtype=np.int64))
    out = torch.empty(ind.shape[0], dtype=torch.float64, device="cuda")
    _lib.check(lib.fm_segment_sums(ind.shape[0], ptr(vals), ptr(ind), ptr(out), stream_ptr()))
    return to_host(out)
