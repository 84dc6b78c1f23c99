"""Device-resident benchmark problems of BASELINE.json (configs 1-5).

Everything is built on the GPU (csrc/fm_prep.cu): mesh, P1 data, Dirichlet
partitions, patch CSR, consistent load and the seeded trial field, then the
evaluation context.  Nothing touches the host except a few counts, so the
config-4/5 sizes (25M / 1.6B tetrahedra) set up in seconds.

Field convention (shared bit-for-bit with the CPU checker in tests): U(seed, k)
= splitmix64(splitmix64(seed) + k) >> 11 * 2^-53 for the global dof k.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import torch

from . import _lib
from ._device import ptr, require_cuda, stream_ptr
from .device import DeviceMesh
from .mesh import _partitions_device, _p1_device
from .models import LameParams, NeoHookean, PLaplaceParams, PLaplacian
from .patches import build_patches_device

E_MOD, NU = 2e8, 0.3


@dataclass
class DeviceProblem:
    name: str
    dm: DeviceMesh
    model: object
    b: torch.Tensor
    v: torch.Tensor
    ne: int
    nn: int
    meta: dict = field(default_factory=dict)


def _finish(name, dim, d, coords, conn, fixed, model, f, field_kind, seed, amp, gid=None,
            tiling=None, meta=None, keep=False):
    lib = require_cuda()
    nn, ne = coords.shape[0], conn.shape[0]
    vol, dphi = _p1_device(dim, coords, conn)
    nd, nm, dd, dm_, dl = _partitions_device(nn, d, fixed)
    prefix, elems, slot = build_patches_device(conn, nm, nn, dim + 1)
    b = torch.empty(nn * d, dtype=torch.float64, device="cuda")
    _lib.check(lib.fm_load_constant(dim, d, nn, ne, ptr(conn), ptr(vol), (C.c_double * d)(*f),
                                    ptr(b), stream_ptr()))
    v = torch.empty(nn * d, dtype=torch.float64, device="cuda")
    if field_kind == "uniform":
        _lib.check(lib.fm_field_uniform(nn * d, ptr(dm_), dm_.numel(), ptr(gid), seed, ptr(v),
                                        stream_ptr()))
    else:
        _lib.check(lib.fm_field_nh(nn, d, ptr(coords), ptr(dm_), dm_.numel(), ptr(gid), seed,
                                   float(amp), ptr(v), stream_ptr()))
    dmesh = DeviceMesh(dim=dim, d=d, coords=coords, conn=conn, volumes=vol, dphi=dphi,
                       nodes_minim=nm, fixed=fixed, p_prefix=prefix, p_elems=elems, p_slot=slot,
                       tiling=tiling)
    meta = dict(meta or {})
    meta.update(nfree_dofs=int(dm_.numel()), patch_rows=int(elems.numel()),
                nodes_dirichlet=int(nd.numel()), dofs_minim=dm_)
    if keep:  # parity tests want the index structures
        meta.update(coords=coords, conn=conn, volumes=vol, dphi=dphi, nodes_minim=nm,
                    dofs_minim=dm_, dofs_minim_local=dl, nodes_dirichlet_idx=nd,
                    dofs_dirichlet=dd, p_prefix=prefix, p_elems=elems, p_slot=slot)
    return DeviceProblem(name, dmesh, model, b, v, ne, nn, meta)


def _predicate(kind, dim, d, coords, fixed, axis=0, c=0.0, tol=1e-9):
    lib = require_cuda()
    matched = C.c_int64(0)
    _lib.check(lib.fm_dirichlet_predicate(kind, dim, d, coords.shape[0], ptr(coords), axis,
                                          float(c), float(tol), None, -1, ptr(fixed),
                                          C.byref(matched), stream_ptr()))
    return matched.value


def lshape(level: int, p: float = 3.0, seed: int = 2109, tiling=None, keep=False):
    """Configs 1/2: bench.py:152-169 (L-shape, full-boundary Dirichlet), f = -10,
    p-Laplace, v = U[0,1) on free dofs.  Config 1 = level 4, config 2 = level 10."""
    lib = require_cuda()
    nn, ne = C.c_int64(), C.c_int64()
    _lib.check(lib.fm_lshape_sizes(level, C.byref(nn), C.byref(ne)))
    coords = torch.empty((nn.value, 2), dtype=torch.float64, device="cuda")
    conn = torch.empty((ne.value, 3), dtype=torch.int64, device="cuda")
    _lib.check(lib.fm_gen_lshape(level, ptr(coords), ptr(conn), stream_ptr()))
    fixed = torch.zeros(nn.value, dtype=torch.uint8, device="cuda")
    _predicate(2, 2, 1, coords, fixed)
    model = PLaplacian(PLaplaceParams(p), dim=2)
    return _finish(f"lshape_l{level}_p{p:g}", 2, 1, coords, conn, fixed, model, [-10.0],
                   "uniform", seed, 0.0, tiling=tiling, keep=keep,
                   meta=dict(level=level, p=p, seed=seed))


def rect(nx: int = 2048, ny: int = 1024, seed: int = 2109, tiling=None, keep=False):
    """Config 3: [0,2]x[0,1], NH 2D (D1 = lambda/2), f = (0,-3.5e7), v = x on x1=0,
    v = x + U[-a,a] with a = 1e-2 h elsewhere."""
    lib = require_cuda()
    coords = torch.empty(((nx + 1) * (ny + 1), 2), dtype=torch.float64, device="cuda")
    conn = torch.empty((2 * nx * ny, 3), dtype=torch.int64, device="cuda")
    _lib.check(lib.fm_gen_rect(nx, ny, 0.0, 2.0, 0.0, 1.0, ptr(coords), ptr(conn), stream_ptr()))
    fixed = torch.zeros(coords.shape[0] * 2, dtype=torch.uint8, device="cuda")
    _predicate(0, 2, 2, coords, fixed)
    model = NeoHookean(LameParams.from_young_poisson(E_MOD, NU), dim=2)
    return _finish(f"rect_{nx}x{ny}", 2, 2, coords, conn, fixed, model, [0.0, -3.5e7], "nh",
                   seed, 1e-2 * (2.0 / nx), tiling=tiling, keep=keep,
                   meta=dict(nx=nx, ny=ny, seed=seed))


def beam(nx: int = 256, ny: int = 128, nz: int = 128, seed: int = 2109, ix0: int = 0,
         ix1: int | None = None, lx=2.0, ly=1.0, lz=1.0, tiling=None, keep=False):
    """Configs 4/5: [0,lx]x[0,ly]x[0,lz] Kuhn beam, NH 3D (D1 = lambda/2),
    f = (0,0,-2.5e7), v = x on x1 = 0.  ``ix0, ix1`` select the x1-slab of
    cubes owned by one rank (global numbering recovered by ``global_node``)."""
    lib = require_cuda()
    ix1 = nx if ix1 is None else ix1
    nxl = ix1 - ix0
    nn = (nxl + 1) * (ny + 1) * (nz + 1)
    coords = torch.empty((nn, 3), dtype=torch.float64, device="cuda")
    conn = torch.empty((6 * nxl * ny * nz, 4), dtype=torch.int64, device="cuda")
    box = (C.c_double * 6)(0.0, lx, 0.0, ly, 0.0, lz)
    _lib.check(lib.fm_gen_beam(nx, ny, nz, box, ix0, ix1, ptr(coords), ptr(conn), stream_ptr()))
    fixed = torch.zeros(nn * 3, dtype=torch.uint8, device="cuda")
    _predicate(0, 3, 3, coords, fixed)
    gid = None
    if nxl != nx:
        gid = global_node(torch.arange(nn, dtype=torch.int64, device="cuda"), nx, ny, ix0, nxl)
    model = NeoHookean(LameParams.from_young_poisson(E_MOD, NU), dim=3)
    return _finish(f"beam_{nx}x{ny}x{nz}[{ix0}:{ix1}]", 3, 3, coords, conn, fixed, model,
                   [0.0, 0.0, -2.5e7], "nh", seed, 1e-2 * (lx / nx), gid=gid, tiling=tiling,
                   keep=keep, meta=dict(nx=nx, ny=ny, nz=nz, ix0=ix0, ix1=ix1, seed=seed))


def global_node(local: torch.Tensor, nx: int, ny: int, ix0: int, nxl: int) -> torch.Tensor:
    """Slab-local node id -> global node id of the (nx, ny, nz) beam."""
    ix = local % (nxl + 1)
    rest = local // (nxl + 1)
    return (ix + ix0) + (nx + 1) * rest


CONFIGS = {
    "cfg1": lambda **kw: lshape(4, 3.0, **kw),
    "cfg2": lambda **kw: lshape(10, 3.0, **kw),
    "cfg2_p1.8": lambda **kw: lshape(10, 1.8, **kw),
    "cfg3": lambda **kw: rect(2048, 1024, **kw),
    "cfg4": lambda **kw: beam(256, 128, 128, **kw),
}
