"""CPU oracle for the P1 energy / gradient hot path — TEST INFRASTRUCTURE ONLY.

This module restates, in plain numpy/scipy, the algorithm of the reference
package ``femmin`` (``/root/reference/pkg/src/femmin``) for the hot path named
in BASELINE.json: mesh generation, P1 basis gradients, Dirichlet partitions,
nodal patches, the batched densities, the energy J, the exact chain-rule
gradient and the nodal-patch central-difference gradient.  Every function cites
the reference ``file:line`` it follows.

It is the *checker*, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` leg may import it.  The product package
(``paper_2109_01158_b200``) never imports this file and has no CPU fallback.

Pinning: ``tests/test_oracle_golden.py`` checks these functions bit-for-bit
against golden vectors produced by the real reference
(``tests/golden/make_golden.py`` imports ``/root/reference/pkg/src``).

Beyond the reference it adds only what the benchmark configs need and the
reference lacks: a parametrised Kuhn beam with free
(nx, ny, nz) and box bounds (restating mesh.py:125-174), a rectangle
(composition of mesh.py:177-192 + 107-122), duck-typed (C1, D1) parameters,
a counter-based splitmix64 field generator shared bit-for-bit with the CUDA
side, and a direct-sum FD variant used to bound GPU FD roundoff.
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass, replace

import numpy as np
import scipy.sparse as sp

# ---------------------------------------------------------------------------
# exceptions (mesh.py:23-28, patches.py:18-19, models.py:16-17)


class OracleMeshError(ValueError):
    pass


class OracleDegenerateElement(OracleMeshError):
    pass


class OraclePatchError(OracleMeshError):
    pass


class OracleInadmissible(ValueError):
    pass


# ---------------------------------------------------------------------------
# containers (mesh.py:31-53, patches.py:22-34)


@dataclass(frozen=True)
class OMesh:
    dim: int
    level: int
    nodes2coord: np.ndarray
    elems2nodes: np.ndarray
    volumes: np.ndarray
    dphi: list
    d: int = 1
    nodes_dirichlet: np.ndarray = None
    nodes_minim: np.ndarray = None
    dofs_dirichlet: np.ndarray = None
    dofs_minim: np.ndarray = None
    dofs_minim_local: np.ndarray = None

    @property
    def nn(self):
        return self.nodes2coord.shape[0]

    @property
    def ne(self):
        return self.elems2nodes.shape[0]


@dataclass(frozen=True)
class OPatches:
    lengths: np.ndarray
    elems: np.ndarray
    slot: np.ndarray      # owner slot per row == argmax(logical) (patches.py:68)
    prefix: np.ndarray

    @property
    def total_rows(self):
        return int(self.elems.shape[0])


# ---------------------------------------------------------------------------
# mesh generation


def p1_gradients(coords: np.ndarray, conn: np.ndarray):
    """Volumes and basis gradients, mesh.py:79-104 (batched LU det / inv)."""
    dim = coords.shape[1]
    X = coords[conn]
    E = X[:, 1:, :] - X[:, :1, :]
    det = np.linalg.det(E)
    vol = det / {1: 1.0, 2: 2.0, 3: 6.0}[dim]
    bad = np.flatnonzero(vol <= 0.0)
    if bad.size:
        raise OracleDegenerateElement(
            f"element {bad[0]} has nonpositive measure {vol[bad[0]]:.3e}")
    inv = np.linalg.inv(E)
    dphi = []
    for m in range(dim):
        g = np.empty((conn.shape[0], dim + 1))
        g[:, 1:] = inv[:, m, :]
        g[:, 0] = -inv[:, m, :].sum(axis=1)
        dphi.append(g)
    return vol, dphi


def _assemble_mesh(dim, level, coords, conn) -> OMesh:
    """mesh.py:107-122: all nodes free until mark_dirichlet."""
    vol, dphi = p1_gradients(coords, conn)
    every = np.arange(coords.shape[0], dtype=np.int64)
    empty = np.empty(0, dtype=np.int64)
    return OMesh(dim, level, coords, conn, vol, dphi, 1,
                 empty, every, empty, every, every)


def grid_triangles(nx: int, ny: int):
    """mesh.py:177-192: two CCW triangles per cell, cell order iy-major."""
    iy, ix = np.divmod(np.arange(nx * ny, dtype=np.int64), nx)
    ll = ix + (nx + 1) * iy
    out = np.empty((nx * ny, 2, 3), dtype=np.int64)
    out[:, 0, 0] = ll
    out[:, 0, 1] = ll + 1
    out[:, 0, 2] = ll + nx + 2
    out[:, 1, 0] = ll
    out[:, 1, 1] = ll + nx + 2
    out[:, 1, 2] = ll + nx + 1
    return out.reshape(-1, 3), ix, iy


def lshape_mesh(level: int) -> OMesh:
    """mesh.py:200-221: (-1,1)^2 minus [0,1]x[-1,0], nodes compressed by
    np.unique rank (mesh.py:195-197)."""
    if level < 0:
        raise ValueError("level must be >= 0")
    n = 2 ** (level + 2)
    xs = np.linspace(-1.0, 1.0, n + 1)
    coords = np.empty(((n + 1) ** 2, 2))
    coords[:, 0] = np.tile(xs, n + 1)
    coords[:, 1] = np.repeat(xs, n + 1)
    tri, ix, iy = grid_triangles(n, n)
    h = 2.0 / n
    drop = ((-1.0 + (ix + 0.5) * h) > 0.0) & ((-1.0 + (iy + 0.5) * h) < 0.0)
    tri = tri.reshape(-1, 2, 3)[~drop].reshape(-1, 3)
    used, inv = np.unique(tri, return_inverse=True)
    return _assemble_mesh(2, level, coords[used], inv.reshape(tri.shape))


def rect_mesh(nx: int, ny: int, x0=0.0, x1=2.0, y0=0.0, y1=1.0) -> OMesh:
    """Config 3 rectangle: np.linspace grid + mesh.py:177-192 + 107-122."""
    xs = np.linspace(x0, x1, nx + 1)
    ys = np.linspace(y0, y1, ny + 1)
    coords = np.empty(((nx + 1) * (ny + 1), 2))
    coords[:, 0] = np.tile(xs, ny + 1)
    coords[:, 1] = np.repeat(ys, nx + 1)
    tri, _, _ = grid_triangles(nx, ny)
    return _assemble_mesh(2, -1, coords, tri)


# Kuhn paths: itertools.permutations(range(3)) order (mesh.py:155);
# odd permutations (slots 1, 2, 5) are negatively oriented on a positive box
# and get local nodes 2 <-> 3 swapped (mesh.py:168-172).
KUHN_PERMS = list(itertools.permutations(range(3)))
KUHN_FLIP = [False, True, True, False, False, True]


def beam_mesh(nx, ny, nz, x0, x1, y0, y1, z0, z1, level=-1, ix0=0, ix1=None) -> OMesh:
    """mesh.py:125-174 with free (nx, ny, nz) and box bounds; optionally only
    the x1-slab of cubes [ix0, ix1) of that grid (slab-local numbering, global
    linspace coordinates)."""
    ix1 = nx if ix1 is None else ix1
    xs = np.linspace(x0, x1, nx + 1)[ix0:ix1 + 1]
    nx = ix1 - ix0
    ys = np.linspace(y0, y1, ny + 1)
    zs = np.linspace(z0, z1, nz + 1)
    N = (nx + 1) * (ny + 1) * (nz + 1)
    coords = np.empty((N, 3))
    coords[:, 0] = np.tile(xs, (ny + 1) * (nz + 1))
    coords[:, 1] = np.tile(np.repeat(ys, nx + 1), nz + 1)
    coords[:, 2] = np.repeat(zs, (nx + 1) * (ny + 1))
    c = np.arange(nx * ny * nz, dtype=np.int64)
    cx = c % nx
    cy = (c // nx) % ny
    cz = c // (nx * ny)
    tets = np.empty((c.size, 6, 4), dtype=np.int64)
    for t, perm in enumerate(KUHN_PERMS):
        off = np.zeros(3, dtype=np.int64)
        cols = [cx + (nx + 1) * (cy + (ny + 1) * cz)]
        for axis in perm:
            off[axis] += 1
            cols.append((cx + off[0]) + (nx + 1) * ((cy + off[1]) + (ny + 1) * (cz + off[2])))
        if KUHN_FLIP[t]:
            cols[2], cols[3] = cols[3], cols[2]
        tets[:, t, :] = np.stack(cols, axis=1)
    return _assemble_mesh(3, level, coords, tets.reshape(-1, 4))


def bar_mesh(lx, ly, lz, level) -> OMesh:
    """generate_bar_mesh_3d (mesh.py:125-174) through the beam restatement."""
    if lx <= 0 or ly <= 0 or lz <= 0:
        raise ValueError("bar dimensions must be positive")
    if level < 1:
        raise ValueError("level must be >= 1")
    s = 2 ** (level - 1)
    return beam_mesh(80 * s, 2 * s, 2 * s, 0.0, lx, -ly / 2, ly / 2,
                     -lz / 2, lz / 2, level)


def mark_dirichlet(mesh: OMesh, fixed: np.ndarray, d: int) -> OMesh:
    """mesh.py:289-322 from the (nn, d) fixed mask the predicates produce."""
    fixed = np.asarray(fixed, dtype=bool).reshape(mesh.nn, d)
    node_fixed = fixed.all(axis=1)
    minim = np.flatnonzero(~node_fixed).astype(np.int64)
    return replace(
        mesh, d=d,
        nodes_dirichlet=np.flatnonzero(node_fixed).astype(np.int64),
        nodes_minim=minim,
        dofs_dirichlet=np.flatnonzero(fixed.ravel()).astype(np.int64),
        dofs_minim=np.flatnonzero(~fixed.ravel()).astype(np.int64),
        dofs_minim_local=np.flatnonzero(~fixed[minim].ravel()).astype(np.int64),
    )


def fixed_mask(mesh: OMesh, regions, d: int) -> np.ndarray:
    """Predicate evaluation part of mesh.py:296-305; regions = [(where, comps)]."""
    fixed = np.zeros((mesh.nn, d), dtype=bool)
    for where, comps in regions:
        mask = np.asarray(where(mesh.nodes2coord), dtype=bool)
        if not mask.any():
            continue
        for j in (range(d) if comps is None else comps):
            fixed[mask, j] = True
    return fixed


def lshape_boundary(level):
    """bench.py:155-166 (tolerance 1e-9)."""
    def on_boundary(x):
        tol = 1e-9
        outer = ((np.abs(x[:, 0] + 1) < tol) | (np.abs(x[:, 0] - 1) < tol)
                 | (np.abs(x[:, 1] + 1) < tol) | (np.abs(x[:, 1] - 1) < tol))
        re = ((np.abs(x[:, 0]) < tol) & (x[:, 1] < tol)) | (
            (np.abs(x[:, 1]) < tol) & (x[:, 0] > -tol))
        return outer | re
    return on_boundary


def left_face(x):
    """x1 = 0 face, the style of bench.py:129 (tol 1e-9)."""
    return x[:, 0] < 1e-9


# ---------------------------------------------------------------------------
# patches (patches.py:37-83)


def build_patches(mesh: OMesh) -> OPatches:
    """patches.py:37-71, keeping (lengths, elems, owner slot, prefix)."""
    ne, nv = mesh.elems2nodes.shape
    node_of = mesh.elems2nodes.ravel()
    elem_of = np.repeat(np.arange(ne, dtype=np.int64), nv)
    slot_of = np.tile(np.arange(nv, dtype=np.int64), ne)
    rank = np.full(mesh.nn, -1, dtype=np.int64)
    rank[mesh.nodes_minim] = np.arange(mesh.nodes_minim.size)
    keys = rank[node_of]
    sel = keys >= 0
    keys, elems, slots = keys[sel], elem_of[sel], slot_of[sel]
    order = np.lexsort((elems, keys))
    keys, elems, slots = keys[order], elems[order], slots[order]
    lengths = np.bincount(keys, minlength=mesh.nodes_minim.size)
    if (lengths == 0).any():
        node = mesh.nodes_minim[np.flatnonzero(lengths == 0)[0]]
        raise OraclePatchError(f"free node {node} has an empty patch")
    return OPatches(lengths.astype(np.int64), elems, slots,
                    np.cumsum(lengths).astype(np.int64))


def prefix_indices(patches: OPatches, d: int) -> np.ndarray:
    """patches.py:74-77."""
    T = patches.total_rows
    return np.concatenate([patches.prefix + b * T for b in range(d)])


def cumsum_segments(values, indx):
    """patches.py:80-83 (global cumsum, then differences)."""
    c = np.cumsum(values)
    return np.diff(c[indx - 1], prepend=0.0)


# ---------------------------------------------------------------------------
# densities (models.py:59-138)


@dataclass(frozen=True)
class LameParams:
    """Duck-typed (C1, D1) holder (configs use D1 = lambda/2)."""
    C1: float
    D1: float

    @classmethod
    def from_E_nu_lambda(cls, E, nu):
        mu = E / (2.0 * (1.0 + nu))
        lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
        return cls(mu / 2.0, lam / 2.0)

    @classmethod
    def from_E_nu_bulk(cls, E, nu):
        """ElasticParams convention, models.py:33-47."""
        mu = E / (2.0 * (1.0 + nu))
        return cls(mu / 2.0, (E / (3.0 * (1.0 - 2.0 * nu))) / 2.0)


def det_batch(F):
    """models.py:59-71 (left-to-right six-term sum in 3D)."""
    if len(F) == 2:
        return F[0][0] * F[1][1] - F[0][1] * F[1][0]
    return (F[0][0] * F[1][1] * F[2][2] + F[0][2] * F[1][0] * F[2][1]
            + F[0][1] * F[1][2] * F[2][0] - F[0][2] * F[1][1] * F[2][0]
            - F[0][1] * F[1][0] * F[2][2] - F[0][0] * F[1][2] * F[2][1])


def cof_batch(F):
    """models.py:74-86."""
    if len(F) == 2:
        return [[F[1][1], -F[1][0]], [-F[0][1], F[0][0]]]
    out = [[None] * 3 for _ in range(3)]
    for j in range(3):
        a, b = [r for r in range(3) if r != j]
        for m in range(3):
            p, q = [c for c in range(3) if c != m]
            minor = F[a][p] * F[b][q] - F[a][q] * F[b][p]
            out[j][m] = minor if (j + m) % 2 == 0 else -minor
    return out


def nh_W(F, prm):
    """models.py:89-100."""
    dim = len(F)
    det = det_batch(F)
    I1 = sum(F[j][m] ** 2 for j in range(dim) for m in range(dim))
    ok = det > 0.0
    ld = np.zeros_like(det)
    np.log(det, out=ld, where=ok)
    W = prm.C1 * (I1 - dim - 2.0 * ld) + prm.D1 * (det - 1.0) ** 2
    if not ok.all():
        W = np.where(ok, W, np.inf)
    return W


def nh_dW(F, prm):
    """models.py:103-120."""
    dim = len(F)
    det = det_batch(F)
    if (det <= 0.0).any():
        raise OracleInadmissible("nonpositive det F in the exact derivative path")
    cof = cof_batch(F)
    dfac = 2.0 * prm.D1 * (det - 1.0)
    inv2 = 2.0 / det
    return [[prm.C1 * (2.0 * F[j][m] - inv2 * cof[j][m]) + dfac * cof[j][m]
             for m in range(dim)] for j in range(dim)]


def plap_W(G, prm):
    """models.py:123-126."""
    n2 = sum(g ** 2 for g in G[0])
    return n2 ** (prm.p / 2.0) / prm.p


def plap_dW(G, prm):
    """models.py:129-138."""
    n2 = sum(g ** 2 for g in G[0])
    if prm.p >= 2.0:
        fac = n2 ** ((prm.p - 2.0) / 2.0)
    else:
        fac = np.zeros_like(n2)
        np.power(n2, (prm.p - 2.0) / 2.0, out=fac, where=n2 > 0.0)
    return [[fac * g for g in G[0]]]


@dataclass(frozen=True)
class PParams:
    p: float


class Model:
    """Model plugin protocol of models.py:141-170: .d .dim .params W dW."""

    def __init__(self, kind: str, params, dim: int):
        self.kind, self.params, self.dim = kind, params, dim
        self.d = dim if kind == "nh" else 1

    def density(self, F):
        return nh_W(F, self.params) if self.kind == "nh" else plap_W(F, self.params)

    def ddensity(self, F):
        return nh_dW(F, self.params) if self.kind == "nh" else plap_dW(F, self.params)


# ---------------------------------------------------------------------------
# assembly (assembly.py:18-120)


def grad_field(dphi, vals):
    """assembly.py:35-49: F[j][m] = einsum('rl,rl->r', v_j, dphi_m)."""
    return [[np.einsum("rl,rl->r", vj, dm) for dm in dphi] for vj in vals]


def element_values(v, d, conn):
    """assembly.py:23-32."""
    V = v.reshape(-1, d)
    return [V[conn, j] for j in range(d)]


def mass_matrix(mesh: OMesh):
    """assembly.py:52-62."""
    nv = mesh.dim + 1
    loc = (np.ones((nv, nv)) + np.eye(nv)) / (nv * (nv + 1))
    vals = mesh.volumes[:, None, None] * loc[None]
    rows = np.repeat(mesh.elems2nodes, nv, axis=1).ravel()
    cols = np.tile(mesh.elems2nodes, (1, nv)).ravel()
    return sp.coo_matrix((vals.ravel(), (rows, cols)), shape=(mesh.nn, mesh.nn)).tocsr()


def load_vector(mesh: OMesh, f, d: int):
    """assembly.py:65-82 (b = M f, interleaved)."""
    M = mass_matrix(mesh)
    f = np.asarray(f, dtype=float)
    Fv = np.broadcast_to(np.atleast_1d(f), (mesh.nn, d)) if f.ndim <= 1 else f
    return np.ascontiguousarray(np.column_stack([M @ Fv[:, j] for j in range(d)])).ravel()


def energy(v, mesh: OMesh, model, b=None):
    """assembly.py:94-106 -> (J, densities)."""
    F = grad_field(mesh.dphi, element_values(v, model.d, mesh.elems2nodes))
    W = model.density(F)
    J = float(mesh.volumes @ W)
    if b is not None:
        J -= float(b @ v)
    return J, W


# ---------------------------------------------------------------------------
# gradients (gradients.py:35-157)


def _rows_to_dofs(blocks, mesh: OMesh, d):
    """gradients.py:68-74."""
    nf = mesh.nodes_minim.size
    out = np.empty(d * nf)
    for j in range(d):
        out[j::d] = blocks[j * nf:(j + 1) * nf]
    return out[mesh.dofs_minim_local]


def _patch_rows(v, mesh: OMesh, P: OPatches, d):
    """gradients.py:59-65 without the patch copies: F on elements copied to rows."""
    F_el = grad_field(mesh.dphi, element_values(v, d, mesh.elems2nodes))
    return F_el, [[fm[P.elems] for fm in fj] for fj in F_el]


def exact_gradient(v, mesh: OMesh, P: OPatches, model, b=None):
    """gradients.py:124-149 (segment sums by global cumsum)."""
    d = model.d
    _, Fp = _patch_rows(v, mesh, P, d)
    dW = model.ddensity(Fp)
    dF = [dm[P.elems, P.slot] for dm in mesh.dphi]          # gradients.py:54-56
    vol = mesh.volumes[P.elems]
    blocks = np.concatenate([vol * sum(dW[j][m] * dF[m] for m in range(mesh.dim))
                             for j in range(d)])
    g = _rows_to_dofs(cumsum_segments(blocks, prefix_indices(P, d)), mesh, d)
    if b is not None:
        g = g - b[mesh.dofs_minim]
    return g


@dataclass(frozen=True)
class RPatches(OPatches):
    """patches.py:22-34 as the reference keeps them: the CSR plus the per-row
    copies of volumes, connectivity, basis gradients and the one-hot owner
    mask (patches.py:61-71).  Used where the reference's per-call WORK must be
    reproduced (bench.py --impl reference), not only its results."""
    volumes: np.ndarray = None
    elems2nodes: np.ndarray = None
    dphi: list = None
    logical: np.ndarray = None


def reference_patches(mesh: OMesh, P: OPatches) -> RPatches:
    """The row copies of patches.py:61-71 on top of the CSR."""
    e2n = mesh.elems2nodes[P.elems]
    owners = mesh.nodes_minim[np.repeat(np.arange(P.lengths.size), P.lengths)]
    return RPatches(P.lengths, P.elems, P.slot, P.prefix, mesh.volumes[P.elems], e2n,
                    [g[P.elems] for g in mesh.dphi], e2n == owners[:, None])


def exact_gradient_femmin(v, mesh: OMesh, RP: RPatches, model, b=None):
    """gradients.py:124-149 doing the reference's per-call work step for step:
    _patch_data (gradients.py:59-65: the element gather and F, the patch-row
    gather v_patches the exact path computes and drops, the F copies to patch
    rows), ddensity on the patch rows, dF_dv_table by the boolean owner mask
    (gradients.py:54-56), the weighted blocks on the stored row volumes and
    the cumsum segment sums (patches.py:80-83).  Same result as
    exact_gradient bit for bit (tests/test_oracle_golden.py)."""
    d, dim = model.d, mesh.dim
    V = v.reshape(-1, d)
    F_el = grad_field(mesh.dphi, [V[mesh.elems2nodes, j] for j in range(d)])
    v_patches = [V[RP.elems2nodes, j] for j in range(d)]  # gradients.py:63 (unused here)
    del v_patches
    Fp = [[fm[RP.elems] for fm in fj] for fj in F_el]
    dW = model.ddensity(Fp)
    dF = [dm[RP.logical] for dm in RP.dphi]
    blocks = np.concatenate([RP.volumes * sum(dW[j][m] * dF[m] for m in range(dim))
                             for j in range(d)])
    g = _rows_to_dofs(cumsum_segments(blocks, prefix_indices(RP, d)), mesh, d)
    if b is not None:
        g = g - b[mesh.dofs_minim]
    return g


def descent_loop(v, mesh: OMesh, P: OPatches, model, b, alpha, iters):
    """Config-5 first-order loop (BASELINE.json configs[4]): ``iters`` times
    J_i = energy(v) (assembly.py:94-106), g = exact_gradient(v)
    (gradients.py:124-149), v[dofs_minim] -= alpha * g.  Returns
    (J history, final v, last g)."""
    v = np.array(v, dtype=np.float64, copy=True)
    Js, g = [], None
    for _ in range(iters):
        Js.append(energy(v, mesh, model, b)[0])
        g = exact_gradient(v, mesh, P, model, b)
        v[mesh.dofs_minim] = v[mesh.dofs_minim] - alpha * g
    return np.array(Js), v, g


def sampled_exact_gradient(v, conn, volumes, dphi, prefix, elems, slot, nodes_minim, d, model,
                           b, dofs_minim, sample):
    """gradients.py:124-149 for a SAMPLE of free dofs only (the
    size-independent check of full-size runs the CPU oracle cannot evaluate
    whole): for free dof q = dofs_minim[sample[i]] (node n, component j), the
    patch rows of n (CSR prefix / elems / slot, patches.py:37-71), F of those
    elements (einsum order), dW (models.py) and
    g = sum_rows vol * sum_m dW[j][m] * dphi[m][row, slot] - b[q], summed in
    patch order (the reference's cumsum differs only by roundoff).
    conn (ne, nv), dphi (dim, ne, nv), prefix inclusive (|M|,)."""
    q = np.asarray(dofs_minim)[np.asarray(sample)]
    node, comp = q // d, q % d
    rank = np.searchsorted(nodes_minim, node)
    lo = np.where(rank > 0, prefix[np.maximum(rank - 1, 0)], 0)
    hi = prefix[rank]
    cnt = hi - lo
    rows = np.concatenate([np.arange(a, z) for a, z in zip(lo, hi)])
    owner = np.repeat(np.arange(q.size), cnt)
    el = elems[rows]
    sl = slot[rows]
    dim = len(dphi)
    F = grad_field([dm[el] for dm in dphi], element_values(v, d, conn[el]))
    dW = model.ddensity(F)
    dF = [dm[el, sl] for dm in dphi]
    jj = comp[owner]
    contrib = np.zeros(rows.size)
    for j in range(d):
        sel = jj == j
        if sel.any():
            contrib[sel] = (volumes[el] * sum(dW[j][m] * dF[m] for m in range(dim)))[sel]
    g = np.zeros(q.size)
    np.add.at(g, owner, contrib)
    return g - (b[q] if b is not None else 0.0)


def _perturbed_row_densities(v, mesh, P, model, eps, with_libm=False):
    """Core of gradients.py:84-121: the d*||T|| densities for each sign
    (-eps first), with G recomputed from perturbed nodal values."""
    d, dim = model.d, mesh.dim
    conn_rows = mesh.elems2nodes[P.elems]
    V = v.reshape(-1, d)
    vrows = [V[conn_rows, j] for j in range(d)]
    _, Fp = _patch_rows(v, mesh, P, d)
    dphi_rows = [dm[P.elems] for dm in mesh.dphi]
    logical = np.zeros(conn_rows.shape, dtype=bool)
    logical[np.arange(conn_rows.shape[0]), P.slot] = True
    out = []
    for s in (-eps, eps):
        veps = [vr + s * logical for vr in vrows]
        G = grad_field(dphi_rows, veps)
        GG = [[np.concatenate([G[j][m] if blk == j else Fp[j][m] for blk in range(d)])
               for m in range(dim)] for j in range(d)]             # gradients.py:35-51
        W = model.density(GG)
        if with_libm:
            # magnitude of the terms W is assembled from: each is rounded at
            # the u level by any evaluation (numpy's, or the GPU's rank-one
            # update of the same invariants, csrc/fm_eval_fd.cu), so two
            # evaluations of one W+- differ by O(u * L):
            # Neo-Hookean C1 (|F|^2 + dim + 2 |log det|) + D1 (det - 1)^2
            # (models.py:89-100); p-Laplace |W| (one pow, models.py:123-126)
            if model.kind == "nh":
                det = det_batch(GG)
                I1 = sum(GG[j][m] ** 2 for j in range(d) for m in range(dim))
                ld = np.abs(np.log(np.where(det > 0, det, 1.0)))
                L = (model.params.C1 * (I1 + dim + 2.0 * ld)
                     + model.params.D1 * (det - 1.0) ** 2)
            else:
                L = np.abs(W)
            out.append((W, L))
        else:
            out.append(W)
    return out


def numeric_gradient(v, mesh: OMesh, P: OPatches, model, b=None, eps=1e-8):
    """gradients.py:84-121, including the offending-dof message (77-81)."""
    d = model.d
    indx = prefix_indices(P, d)
    vols = np.tile(mesh.volumes[P.elems], d)
    sums = []
    for W in _perturbed_row_densities(v, mesh, P, model, eps):
        ok = np.isfinite(W)
        if not ok.all():
            row = int(np.flatnonzero(~ok)[0])
            T = P.total_rows
            i = int(np.searchsorted(P.prefix, row % T, side="right"))
            raise OracleInadmissible(
                f"perturbed state inadmissible at dof {int(d * mesh.nodes_minim[i] + row // T)}")
        sums.append(cumsum_segments(vols * W, indx))
    g = _rows_to_dofs((sums[1] - sums[0]) / (2.0 * eps), mesh, d)
    if b is not None:
        g = g - b[mesh.dofs_minim]
    return g


def numeric_gradient_direct(v, mesh: OMesh, P: OPatches, model, b=None, eps=1e-8):
    """Same central differences with per-patch sequential sums instead of the
    global cumsum; also returns a per-dof roundoff scale
    u * sum_patch vol*(|W+| + |W-| + L+ + L-) / (2 eps) used as the FD parity
    bound, L the magnitude of the terms W+- is assembled from (their rounding
    is what two evaluations of the same W+- may differ by)."""
    d = model.d
    (Wm, Lm), (Wp, Lp) = _perturbed_row_densities(v, mesh, P, model, eps, with_libm=True)
    T = P.total_rows
    vol = mesh.volumes[P.elems]
    starts = np.concatenate([[0], P.prefix[:-1]])
    Sp, Sm, Sa = [], [], []
    for j in range(d):
        sl = slice(j * T, (j + 1) * T)
        wp = vol * Wp[sl]
        wm = vol * Wm[sl]
        Sp.append(np.add.reduceat(wp, starts))
        Sm.append(np.add.reduceat(wm, starts))
        Sa.append(np.add.reduceat(np.abs(wp) + np.abs(wm) + vol * (Lp[sl] + Lm[sl]), starts))
    g = _rows_to_dofs((np.concatenate(Sp) - np.concatenate(Sm)) / (2.0 * eps), mesh, d)
    scale = _rows_to_dofs(np.concatenate(Sa) * np.finfo(float).eps / (2.0 * eps), mesh, d)
    if b is not None:
        g = g - b[mesh.dofs_minim]
    return g, scale


def exact_gradient_loop(v, mesh: OMesh, model):
    """Element-loop oracle in the spirit of test_gradients.py:133-155:
    per free node, sum over incident elements of vol * dW : grad phi."""
    d, dim = model.d, mesh.dim
    F = grad_field(mesh.dphi, element_values(v, d, mesh.elems2nodes))
    dW = model.ddensity(F)
    nv = dim + 1
    acc = np.zeros((mesh.nn, d))
    for j in range(d):
        for s in range(nv):
            c = mesh.volumes * sum(dW[j][m] * mesh.dphi[m][:, s] for m in range(dim))
            np.add.at(acc[:, j], mesh.elems2nodes[:, s], c)
    return acc.ravel()[mesh.dofs_minim]


# ---------------------------------------------------------------------------
# seeded fields: counter-based splitmix64 (identical on the CUDA side)

_GOLD = np.uint64(0x9E3779B97F4A7C15)


def splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (x + _GOLD).astype(np.uint64)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def uniform01(seed: int, idx: np.ndarray) -> np.ndarray:
    """U[0,1) with 53 bits: splitmix64(splitmix64(seed) + idx) >> 11 * 2^-53."""
    base = splitmix64(np.array([seed], dtype=np.uint64))[0]
    with np.errstate(over="ignore"):
        z = splitmix64((np.asarray(idx, dtype=np.uint64) + base).astype(np.uint64))
    return (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def field_plap(mesh: OMesh, seed: int) -> np.ndarray:
    """Configs 1/2: U[0,1) on free dofs, 0 on Dirichlet dofs (d = 1)."""
    v = np.zeros(mesh.nn)
    v[mesh.dofs_minim] = uniform01(seed, mesh.dofs_minim)
    return v


def field_nh(mesh: OMesh, seed: int, amp: float) -> np.ndarray:
    """Configs 3-5: v = x + amp*(2U-1) on free dofs, v = x on fixed dofs."""
    v = np.ascontiguousarray(mesh.nodes2coord).ravel().copy()
    dof = mesh.dofs_minim
    v[dof] = v[dof] + amp * (2.0 * uniform01(seed, dof) - 1.0)
    return v


# ---------------------------------------------------------------------------
# benchmark problems (BASELINE.json configs)

E_MOD, NU = 2e8, 0.3


def problem_lshape(level: int, p: float, seed: int = 2109):
    """Configs 1/2: bench.py:152-169 mesh + Dirichlet, f = -10, U[0,1) field."""
    m = lshape_mesh(level)
    m = mark_dirichlet(m, fixed_mask(m, [(lshape_boundary(level), None)], 1), 1)
    b = load_vector(m, -10.0, 1)
    return m, Model("plap", PParams(p), 2), b, field_plap(m, seed)


def problem_rect(nx: int, ny: int, seed: int = 2109):
    """Config 3: [0,2]x[0,1], NH 2D, D1 = lambda/2, f = (0,-3.5e7), v=x on x1=0."""
    m = rect_mesh(nx, ny, 0.0, 2.0, 0.0, 1.0)
    m = mark_dirichlet(m, fixed_mask(m, [(left_face, None)], 2), 2)
    b = load_vector(m, (0.0, -3.5e7), 2)
    model = Model("nh", LameParams.from_E_nu_lambda(E_MOD, NU), 2)
    return m, model, b, field_nh(m, seed, 1e-2 * (2.0 / nx))


def problem_beam(nx: int, ny: int, nz: int, seed: int = 2109, lx=2.0, ly=1.0, lz=1.0,
                 ix0: int = 0, ix1: int | None = None):
    """Configs 4/5: [0,lx]x[0,ly]x[0,lz] Kuhn beam, NH 3D, f = (0,0,-2.5e7).
    With (ix0, ix1): the slab of one rank of the x1 partition; its
    load vector sums only the slab's elements and the field draws the global
    dof hash."""
    ix1 = nx if ix1 is None else ix1
    m = beam_mesh(nx, ny, nz, 0.0, lx, 0.0, ly, 0.0, lz, ix0=ix0, ix1=ix1)
    m = mark_dirichlet(m, fixed_mask(m, [(left_face, None)], 3), 3)
    b = load_vector(m, (0.0, 0.0, -2.5e7), 3)
    model = Model("nh", LameParams.from_E_nu_lambda(E_MOD, NU), 3)
    nxl = ix1 - ix0
    local = np.arange(m.nn, dtype=np.int64)
    gid = (local % (nxl + 1) + ix0) + (nx + 1) * (local // (nxl + 1))
    v = np.ascontiguousarray(m.nodes2coord).ravel().copy()
    dof = m.dofs_minim
    gdof = 3 * gid[dof // 3] + dof % 3
    v[dof] = v[dof] + 1e-2 * (lx / nx) * (2.0 * uniform01(seed, gdof) - 1.0)
    return m, model, b, v
