"""Structured simplex meshes, P1 element data and Dirichlet partitions (GPU).

Mirror of ``/root/reference/pkg/src/femmin/mesh.py``: same ``Mesh`` dataclass,
generator names, exceptions and index conventions (0-based int64, x-fastest
lexicographic nodes, interleaved dofs).  The generators, the P1 gradients and
the node/dof partitions run as CUDA kernels (csrc/fm_prep.cu); the returned
arrays are bit-exact with the reference for every index structure and for
coordinates.  The device copies stay attached to the returned Mesh so a later
evaluation context does not upload them again.
"""

from __future__ import annotations

import ctypes as C
import logging
from dataclasses import dataclass, field, replace
from typing import Callable, Sequence

import numpy as np
import torch

from . import _lib
from ._device import ptr, require_cuda, stream_ptr, to_dev, to_host
from .device import attach, attached

logger = logging.getLogger(__name__)

_EMPTY = np.empty(0, dtype=np.int64)


class MeshError(ValueError):
    pass


class DegenerateElementError(MeshError):
    """A simplex with zero or negative measure was encountered (mesh.py:27-28)."""


@dataclass(frozen=True)
class Mesh:
    """mesh.py:31-53."""

    dim: int
    level: int
    nodes2coord: np.ndarray
    elems2nodes: np.ndarray
    volumes: np.ndarray
    dphi: list
    d: int = 1
    nodes_dirichlet: np.ndarray = field(default_factory=lambda: _EMPTY)
    nodes_minim: np.ndarray = field(default_factory=lambda: _EMPTY)
    dofs_dirichlet: np.ndarray = field(default_factory=lambda: _EMPTY)
    dofs_minim: np.ndarray = field(default_factory=lambda: _EMPTY)
    dofs_minim_local: np.ndarray = field(default_factory=lambda: _EMPTY)

    @property
    def nn(self) -> int:
        return self.nodes2coord.shape[0]

    @property
    def ne(self) -> int:
        return self.elems2nodes.shape[0]


@dataclass(frozen=True)
class DirichletRegion:
    """mesh.py:56-68: coordinate predicate, fixed components, optional values."""

    where: Callable[[np.ndarray], np.ndarray]
    components: tuple | None = None
    value: Callable | None = None


@dataclass(frozen=True)
class DirichletSpec:
    regions: tuple

    def __init__(self, regions: Sequence[DirichletRegion]):
        object.__setattr__(self, "regions", tuple(regions))


# --------------------------------------------------------------------------
# device helpers


def _p1_device(dim, coords_d, conn_d):
    lib = require_cuda()
    ne = conn_d.shape[0]
    vol = torch.empty(ne, dtype=torch.float64, device="cuda")
    dphi = torch.empty((dim, ne, dim + 1), dtype=torch.float64, device="cuda")
    bad = C.c_int64(-1)
    _lib.check(lib.fm_p1_gradients(dim, coords_d.shape[0], ne, ptr(coords_d), ptr(conn_d),
                                   ptr(vol), ptr(dphi), C.byref(bad), stream_ptr()))
    return vol, dphi


def _mesh_from_device(dim, level, coords_d, conn_d) -> Mesh:
    """_make_mesh (mesh.py:107-122): P1 data on the GPU, all nodes free."""
    vol_d, dphi_d = _p1_device(dim, coords_d, conn_d)
    nn = coords_d.shape[0]
    every = np.arange(nn, dtype=np.int64)
    dphi_h = to_host(dphi_d)
    m = Mesh(dim=dim, level=level, nodes2coord=to_host(coords_d), elems2nodes=to_host(conn_d),
             volumes=to_host(vol_d), dphi=[dphi_h[k] for k in range(dim)],
             nodes_dirichlet=_EMPTY, nodes_minim=every, dofs_dirichlet=_EMPTY,
             dofs_minim=every, dofs_minim_local=every)
    attach(m, coords=coords_d, conn=conn_d, volumes=vol_d, dphi=dphi_d)
    return m


def compute_p1_gradients(nodes2coord: np.ndarray, elems2nodes: np.ndarray):
    """mesh.py:79-104 -> (volumes, dphi); DegenerateElementError on vol <= 0."""
    coords_d = to_dev(np.asarray(nodes2coord, dtype=np.float64))
    conn_d = to_dev(np.asarray(elems2nodes, dtype=np.int64))
    dim = coords_d.shape[1]
    vol_d, dphi_d = _p1_device(dim, coords_d, conn_d)
    dphi_h = to_host(dphi_d)
    return to_host(vol_d), [dphi_h[k] for k in range(dim)]


def _make_mesh(dim, level, nodes2coord, elems2nodes) -> Mesh:
    return _mesh_from_device(dim, level, to_dev(np.asarray(nodes2coord, dtype=np.float64)),
                             to_dev(np.asarray(elems2nodes, dtype=np.int64)))


# --------------------------------------------------------------------------
# generators


def generate_beam_mesh_3d(nx: int, ny: int, nz: int, box=(0.0, 2.0, 0.0, 1.0, 0.0, 1.0),
                          level: int = -1) -> Mesh:
    """Kuhn beam with free (nx, ny, nz) cubes on box (x0,x1,y0,y1,z0,z1);
    generate_bar_mesh_3d (mesh.py:125-174) is the special case below."""
    lib = require_cuda()
    box = [float(b) for b in box]
    if not (box[1] > box[0] and box[3] > box[2] and box[5] > box[4]):
        raise ValueError("bar dimensions must be positive")
    nn = (nx + 1) * (ny + 1) * (nz + 1)
    coords = torch.empty((nn, 3), dtype=torch.float64, device="cuda")
    conn = torch.empty((6 * nx * ny * nz, 4), dtype=torch.int64, device="cuda")
    _lib.check(lib.fm_gen_beam(nx, ny, nz, (C.c_double * 6)(*box), 0, nx, ptr(coords),
                               ptr(conn), stream_ptr()))
    return _mesh_from_device(3, level, coords, conn)


def generate_bar_mesh_3d(lx: float, ly: float, lz: float, level: int) -> Mesh:
    """mesh.py:125-174: 80*2^(l-1) x 2*2^(l-1) x 2*2^(l-1) cubes on
    (0,lx) x (-ly/2,ly/2) x (-lz/2,lz/2)."""
    if lx <= 0 or ly <= 0 or lz <= 0:
        raise ValueError("bar dimensions must be positive")
    if level < 1:
        raise ValueError("level must be >= 1")
    s = 2 ** (level - 1)
    return generate_beam_mesh_3d(80 * s, 2 * s, 2 * s,
                                 (0.0, lx, -ly / 2, ly / 2, -lz / 2, lz / 2), level)


def generate_lshape_mesh_2d(level: int) -> Mesh:
    """mesh.py:200-221: (-1,1)^2 minus [0,1]x[-1,0], h = 2^-(level+1)."""
    if level < 0:
        raise ValueError("level must be >= 0")
    lib = require_cuda()
    nn, ne = C.c_int64(), C.c_int64()
    _lib.check(lib.fm_lshape_sizes(level, C.byref(nn), C.byref(ne)))
    coords = torch.empty((nn.value, 2), dtype=torch.float64, device="cuda")
    conn = torch.empty((ne.value, 3), dtype=torch.int64, device="cuda")
    _lib.check(lib.fm_gen_lshape(level, ptr(coords), ptr(conn), stream_ptr()))
    return _mesh_from_device(2, level, coords, conn)


def generate_rect_mesh_2d(nx: int, ny: int, box=(0.0, 2.0, 0.0, 1.0)) -> Mesh:
    """Config-3 rectangle: linspace grid + _grid_triangles (mesh.py:177-192)."""
    lib = require_cuda()
    coords = torch.empty(((nx + 1) * (ny + 1), 2), dtype=torch.float64, device="cuda")
    conn = torch.empty((2 * nx * ny, 3), dtype=torch.int64, device="cuda")
    _lib.check(lib.fm_gen_rect(nx, ny, *[float(b) for b in box], ptr(coords), ptr(conn),
                               stream_ptr()))
    return _mesh_from_device(2, -1, coords, conn)


# --------------------------------------------------------------------------
# Dirichlet partitions


def _partitions_device(nn: int, d: int, fixed_d: torch.Tensor):
    lib = require_cuda()
    out = [torch.empty(n, dtype=torch.int64, device="cuda") for n in (nn, nn, nn * d, nn * d)]
    loc = torch.empty(nn * d, dtype=torch.int64, device="cuda")
    counts = (C.c_int64 * 5)()
    _lib.check(lib.fm_mark_dirichlet(nn, d, ptr(fixed_d), *[ptr(t) for t in out], ptr(loc),
                                     counts, stream_ptr()))
    nd, nm, dd, dm, dl = list(counts)
    return out[0][:nd], out[1][:nm], out[2][:dd], out[3][:dm], loc[:dl]


def mark_dirichlet(mesh: Mesh, spec: DirichletSpec, d: int) -> Mesh:
    """mesh.py:289-322.  The region predicates are user callables evaluated on
    the coordinates; the node/dof partitions are computed on the GPU."""
    nn = mesh.nn
    fixed = np.zeros((nn, d), dtype=bool)
    for region in spec.regions:
        mask = np.asarray(region.where(mesh.nodes2coord), dtype=bool)
        if not mask.any():
            logger.warning("Dirichlet region matched no nodes")
            continue
        comps = range(d) if region.components is None else region.components
        for j in comps:
            fixed[mask, j] = True
    fixed_d = to_dev(fixed.astype(np.uint8).ravel())
    nd, nm, dd, dm, dl = _partitions_device(nn, d, fixed_d)
    out = replace(mesh, d=d, nodes_dirichlet=to_host(nd), nodes_minim=to_host(nm),
                  dofs_dirichlet=to_host(dd), dofs_minim=to_host(dm),
                  dofs_minim_local=to_host(dl))
    dev = attached(mesh)
    if dev:
        attach(out, **{k: dev[k] for k in ("coords", "conn", "volumes", "dphi") if k in dev},
               fixed=fixed_d, nodes_minim=nm, dofs_minim=dm)
    return out


def dirichlet_values(mesh: Mesh, spec: DirichletSpec, d: int, t=None) -> np.ndarray:
    """mesh.py:325-341: prescribed values on all dofs (free entries zero);
    evaluates the user's value callables (caller-side glue, not the hot path)."""
    values = np.zeros((mesh.nn, d))
    for region in spec.regions:
        mask = np.asarray(region.where(mesh.nodes2coord), dtype=bool)
        if not mask.any():
            continue
        comps = list(range(d)) if region.components is None else list(region.components)
        idx = np.ix_(np.flatnonzero(mask), comps)
        if region.value is not None:
            values[idx] = np.asarray(region.value(mesh.nodes2coord[mask], t), dtype=float)
        else:
            values[idx] = 0.0
    return values.ravel()
