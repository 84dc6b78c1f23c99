"""Multi-GPU x1-slab partition of the Kuhn beam (configs 4/5).

Each rank generates and evaluates its own slab of cubes ix in [ix0, ix1)
(``problems.beam(..., ix0=, ix1=)``): elements are disjoint, the nodes of the
interface planes x = xs[ix0] and x = xs[ix1] are shared with the neighbours.
Because J, the consistent load b and the element contributions to grad J are
all sums over elements, each rank's slab-local results are exact partial sums:

* J       = sum over ranks of the local J (elastic part and b.v both split by
            elements) -> all-gather of 3 doubles, summed by one fixed reduction
            on every rank, so every rank holds the same bits;
* grad J  = local value at interior nodes; at an interface node the sum of the
            two neighbours' partials, exchanged as one plane buffer
            (ny+1)(nz+1)*3 doubles per side over NCCL send/recv and added as
            own + received (a + b == b + a, so both copies are bitwise equal).

The descent update of config 5 then needs no further exchange.
"""

from __future__ import annotations

import os
import weakref

import torch
import torch.distributed as dist


def slab_range(nx: int, rank: int, world: int) -> tuple[int, int]:
    """Cubes [ix0, ix1) of rank ``rank`` (balanced contiguous x1-slabs)."""
    return nx * rank // world, nx * (rank + 1) // world


def plane_nodes(ixl: int, nxl: int, ny: int, nz: int, device=None) -> torch.Tensor:
    """Slab-local node ids of the x-plane ixl (0 <= ixl <= nxl), (iy, iz) order."""
    k = torch.arange((ny + 1) * (nz + 1), dtype=torch.int64, device=device)
    return ixl + (nxl + 1) * k


def plane_dof_positions(nodes: torch.Tensor, d: int, dofs_minim: torch.Tensor) -> torch.Tensor:
    """Positions of the nodes' d dofs (node-major) in the restricted gradient."""
    dofs = (nodes[:, None] * d + torch.arange(d, device=nodes.device)[None]).reshape(-1)
    pos = torch.searchsorted(dofs_minim, dofs)
    if not torch.equal(dofs_minim[pos.clamp(max=dofs_minim.numel() - 1)], dofs):
        raise ValueError("interface plane holds Dirichlet dofs; slabs must not cut x1 = 0")
    return pos


class NativeSlab:
    """The exchange through the C ABI (include/femmin_b200.h fm_slab_*): its
    own NCCL communicator (unique id from rank 0, broadcast over the torch
    process group), the plane positions uploaded once."""

    def __init__(self, left, right, n_plane, rank, world, group=None):
        import ctypes as C

        from . import _lib
        from ._device import ptr
        self._lib = _lib
        self.lib = _lib.load()
        uid = (C.c_char * 128)()
        if rank == 0:
            _lib.check(self.lib.fm_comm_unique_id(uid), "fm_comm_unique_id")
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=0, group=group)
        uid = (C.c_char * 128).from_buffer_copy(box[0])
        self.left = left.contiguous() if left is not None else None
        self.right = right.contiguous() if right is not None else None
        for plane in (self.left, self.right):
            if plane is not None and plane.numel() != n_plane:
                raise ValueError("interface plane size mismatch")
        h = C.c_void_p()
        _lib.check(self.lib.fm_slab_create(uid, rank, world, int(n_plane), ptr(self.left),
                                           ptr(self.right), C.byref(h)), "fm_slab_create")
        self._h = h
        self._fin = weakref.finalize(self, self.lib.fm_slab_destroy, h)

    def reduce(self, g, J):
        from ._device import ptr, stream_ptr
        self._lib.check(self.lib.fm_slab_reduce(self._h, ptr(g), ptr(J), stream_ptr()),
                        "fm_slab_reduce")


class SlabExchange:
    """Reduction of slab-local (J, grad J) partials across the x1-slab ranks."""

    def __init__(self, nx, ny, nz, ix0, ix1, d, dofs_minim, rank, world, group=None):
        nxl = ix1 - ix0
        dev = dofs_minim.device
        left = (plane_dof_positions(plane_nodes(0, nxl, ny, nz, dev), d, dofs_minim)
                if rank > 0 else None)
        right = (plane_dof_positions(plane_nodes(nxl, nxl, ny, nz, dev), d, dofs_minim)
                 if rank < world - 1 else None)
        self._setup(left, right, (ny + 1) * (nz + 1) * d, dev, rank, world, group)

    @classmethod
    def from_positions(cls, left, right, n, device, rank, world, group=None):
        """The exchange for given plane positions in g (``left`` / ``right``:
        device int64 (n,) or None where there is no neighbour)."""
        ex = cls.__new__(cls)
        ex._setup(left, right, n, device, rank, world, group)
        return ex

    def _setup(self, left, right, n, dev, rank, world, group):
        self.rank, self.world, self.group = rank, world, group
        self.left, self.right = left, right
        # both planes packed / added back with one launch each: positions
        # [left | right], send and receive buffers with the same layout
        planes = [p for p in (self.left, self.right) if p is not None]
        self.pos = torch.cat(planes) if planes else None
        self.n = n
        self.send = torch.empty(len(planes) * n, dtype=torch.float64, device=dev)
        self.recv = torch.empty_like(self.send)
        self.jall = torch.empty((world, 3), dtype=torch.float64, device=dev)
        # NCCL moves device buffers; a gloo group (CPU tests, or the one-GPU
        # functional smoke test of the multi-rank bench) needs host copies
        backend = dist.get_backend(group)
        self.host = dev.type == "cuda" and backend != "nccl"
        # with NCCL the exchange runs in the C ABI (fm_slab_reduce: pack, one
        # grouped NCCL launch for both planes and the J all-gather, unpack);
        # FM_SLAB_TORCH=1 keeps the torch.distributed path below
        self.native = None
        if (dev.type == "cuda" and backend == "nccl"
                and os.environ.get("FM_SLAB_TORCH", "0") != "1"):
            self.native = NativeSlab(self.left, self.right, n, rank, world, group)

    @classmethod
    def from_problem(cls, pr, rank, world, group=None):
        if isinstance(pr.dm, SlabStack):
            st = pr.dm
            return cls.from_positions(st.outer_left if rank > 0 else None,
                                      st.outer_right if rank < world - 1 else None,
                                      st.n_plane, st.device, rank, world, group)
        mt = pr.meta
        return cls(mt["nx"], mt["ny"], mt["nz"], mt["ix0"], mt["ix1"], pr.dm.d,
                   mt["dofs_minim"], rank, world, group)

    def reduce(self, g: torch.Tensor | None, J: torch.Tensor | None = None):
        """In place: g += neighbours' interface partials; J <- global J
        (the all-gathered per-rank partials summed by one fixed reduction, the
        same on every rank).  Either may be None."""
        if self.native is not None:
            self.native.reduce(g, J)
            return g, J
        if g is not None and self.pos is not None:
            torch.index_select(g, 0, self.pos, out=self.send)
            send = self.send.cpu() if self.host else self.send
            recv = self.recv.cpu() if self.host else self.recv
            ops, k = [], 0
            for peer, plane in ((self.rank - 1, self.left), (self.rank + 1, self.right)):
                if plane is None:
                    continue
                sl = slice(k * self.n, (k + 1) * self.n)
                ops += [dist.P2POp(dist.isend, send[sl], peer, self.group),
                        dist.P2POp(dist.irecv, recv[sl], peer, self.group)]
                k += 1
            for req in dist.batch_isend_irecv(ops):
                req.wait()
            if recv is not self.recv:
                self.recv.copy_(recv)
            g.index_add_(0, self.pos, self.recv)
        if J is not None:
            if self.host:
                ja = self.jall.cpu()
                dist.all_gather_into_tensor(ja, J.reshape(1, 3).cpu(), group=self.group)
                self.jall.copy_(ja)
            else:
                dist.all_gather_into_tensor(self.jall, J.reshape(1, 3).contiguous(),
                                            group=self.group)
            torch.sum(self.jall, 0, out=J)
        return g, J


def stack_parts(ne: int, max_elems: int) -> int:
    """Sub-slabs needed so that none holds more than ``max_elems`` elements."""
    return max(1, -(-int(ne) // int(max_elems)))


def stack_ranges(ix0: int, ix1: int, parts: int) -> list[tuple[int, int]]:
    """Cube ranges of the sub-slabs of [ix0, ix1): near-equal, each sized so
    that its free node layers fill whole tile boxes along x1 (8 layers: n + 1
    layers for n cubes, n for the slab at x1 = 0 whose first layer is
    Dirichlet); the last sub-slab takes the remainder.  Measured on the cfg5
    2-way share (6 sub-slabs): 30.7 ms with these cuts, 30.8 ms with an even
    split into 85 / 86 cubes, 32.4 ms with cuts on multiples of 8 cubes (a
    single leftover node layer per sub-slab)."""
    nxl = ix1 - ix0
    parts = max(1, min(int(parts), nxl))
    if nxl < 16 * parts:  # small slabs: an even split
        return [(ix0 + nxl * k // parts, ix0 + nxl * (k + 1) // parts) for k in range(parts)]
    cuts, a = [ix0], ix0
    for k in range(parts - 1):
        want = ix0 + round(nxl * (k + 1) / parts) - a
        r = 0 if a == 0 else 7  # cubes mod 8 that fill whole boxes
        n = max(1, want + ((r - want) % 8 if (r - want) % 8 <= 4 else (r - want) % 8 - 8))
        n = min(n, ix1 - a - (parts - 1 - k))  # leave at least a cube per later part
        a += n
        cuts.append(a)
    cuts.append(ix1)
    return [(cuts[k], cuts[k + 1]) for k in range(parts)]


class SlabStack:
    """A rank's x1-slab [ix0, ix1) of the Kuhn beam held as K sub-slab
    evaluation contexts on ONE GPU, for slabs too large for one context
    (config 5 at 2 GPUs: 805 M tetrahedra per rank; a context indexes its
    patch rows with 32-bit integers and its build peaks at ~450 B per
    element).  Sub-slab k covers the cubes [a_k, a_{k+1}); consecutive
    sub-slabs share one node plane, exactly like neighbouring ranks, and their
    partials there are summed on the device (``fm_stack_reduce``: own +
    neighbour stored to both copies, J summed in sub-slab order).  The
    contexts are built one after another, each from its own generated
    sub-mesh whose reference-format arrays are released before the next build,
    so the device holds K compact contexts, never K sets of build inputs.

    Duck-types the ``DeviceMesh`` calls the benchmark makes (exact_gradient,
    energy, numeric_gradient, descent, check, launches, stats) on the
    concatenated vectors: the field / load ``V`` / ``B`` are the sub-slabs'
    (nn_k d) blocks back to back, the gradient ``G`` their (nfree_dofs_k)
    blocks.  The rank's outer interface planes (``outer_left`` /
    ``outer_right``, positions in G) go to ``SlabExchange.from_positions``.
    """

    def __init__(self, nx, ny, nz, ix0, ix1, parts, seed=2109, tiling=None):
        from . import problems
        dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        self.nx, self.ny, self.nz, self.ix0, self.ix1 = nx, ny, nz, ix0, ix1
        nxl = ix1 - ix0
        parts = max(1, min(int(parts), nxl))
        self.ranges = stack_ranges(ix0, ix1, parts)
        d = 3
        self.dim, self.d = 3, d
        nn_k = [(z - a + 1) * (ny + 1) * (nz + 1) for a, z in self.ranges]
        self.voff = [0]
        for n in nn_k:
            self.voff.append(self.voff[-1] + n * d)
        self.V = torch.empty(self.voff[-1], dtype=torch.float64, device=dev)
        self.B = torch.empty(self.voff[-1], dtype=torch.float64, device=dev)
        self.n_plane = (ny + 1) * (nz + 1) * d
        self.dms, lefts, rights, nfd = [], [], [], []
        self.model = None
        for k, (a, z) in enumerate(self.ranges):
            pr = problems.beam(nx, ny, nz, seed=seed, ix0=a, ix1=z, tiling=tiling)
            self.model = pr.model
            self.V[self.voff[k]:self.voff[k + 1]].copy_(pr.v)
            self.B[self.voff[k]:self.voff[k + 1]].copy_(pr.b)
            dmin = pr.meta["dofs_minim"]
            lefts.append(plane_dof_positions(plane_nodes(0, z - a, ny, nz, dev), d, dmin)
                         if (k > 0 or a > 0) else None)
            rights.append(plane_dof_positions(plane_nodes(z - a, z - a, ny, nz, dev), d, dmin)
                          if (k < parts - 1 or z < nx) else None)
            nfd.append(pr.dm.nfree_dofs)
            self.dms.append(pr.dm)
            del pr, dmin
        self.goff = [0]
        for n in nfd:
            self.goff.append(self.goff[-1] + n)
        # interface dofs between consecutive sub-slabs, positions in G
        if parts > 1:
            self.pa = torch.cat([rights[k] + self.goff[k] for k in range(parts - 1)])
            self.pb = torch.cat([lefts[k + 1] + self.goff[k + 1] for k in range(parts - 1)])
        else:
            self.pa = self.pb = None
        self.outer_left = lefts[0] if lefts[0] is not None else None
        self.outer_right = (rights[-1] + self.goff[-2]) if rights[-1] is not None else None
        self.K = parts
        self.Jk = torch.zeros((parts, 3), dtype=torch.float64, device=dev)
        self.ne = sum(m.ne for m in self.dms)
        self.nn = self.voff[-1] // d
        self.nfree_dofs = self.goff[-1]
        st = [m.stats for m in self.dms]
        self.stats = dict(st[0])
        for key in ("n_tiles", "n_orphan_tiles", "tile_elems_total", "node_entries_total",
                    "bytes_device", "cross_entries", "dict_tiles"):
            self.stats[key] = sum(x[key] for x in st)
        for key in ("max_tile_elems", "max_tile_entries", "entry_cap", "closure_cap"):
            self.stats[key] = max(x[key] for x in st)
        self.stats["redundancy"] = self.stats["tile_elems_total"] / self.ne
        self.stats["sub_slabs"] = parts
        self._lib = self.dms[0]._lib
        self._own_launches = 0
        self._kev = None  # armed per-sub tile-kernel events (time_next)
        self._kms = []

    # per-sub views of the concatenated vectors
    def _v(self, X, k):
        return X[self.voff[k]:self.voff[k + 1]] if X is not None else None

    def _g(self, G, k):
        return G[self.goff[k]:self.goff[k + 1]]

    def _reduce(self, G, J):
        from . import _lib
        from ._device import ptr, stream_ptr
        n = self.pa.numel() if (G is not None and self.pa is not None) else 0
        if n == 0 and J is None:
            return
        _lib.check(self._lib.fm_stack_reduce(n, ptr(self.pa) if n else None,
                                             ptr(self.pb) if n else None,
                                             ptr(G) if n else None, ptr(self.Jk), self.K,
                                             ptr(J), stream_ptr()), "fm_stack_reduce")
        self._own_launches += 1

    def _arm(self, k):
        if self._kev is not None:
            self.dms[k].time_next(*self._kev[k])

    def _collect(self):
        if self._kev is not None:
            self._pending.append(self._kev)
            self._kev = None

    def exact_gradient(self, v, model, b=None, g=None, J=None):
        if g is None:
            g = torch.empty(self.nfree_dofs, dtype=torch.float64, device=self.device)
        for k, m in enumerate(self.dms):
            self._arm(k)
            m.exact_gradient(self._v(v, k), model, self._v(b, k), g=self._g(g, k),
                             J=self.Jk[k] if J is not None else None)
        self._collect()
        self._reduce(g, J)
        return g

    def energy(self, v, model, b=None, out=None):
        out = torch.empty(3, dtype=torch.float64, device=self.device) if out is None else out
        for k, m in enumerate(self.dms):
            m.energy(self._v(v, k), model, self._v(b, k), out=self.Jk[k])
        self._reduce(None, out)
        return out

    def numeric_gradient(self, v, model, b=None, eps=1e-8, g=None):
        if g is None:
            g = torch.empty(self.nfree_dofs, dtype=torch.float64, device=self.device)
        for k, m in enumerate(self.dms):
            self._arm(k)
            m.numeric_gradient(self._v(v, k), model, self._v(b, k), eps, g=self._g(g, k))
        self._collect()
        self._reduce(g, None)
        return g

    def descent_step(self, v, g, alpha):
        for k, m in enumerate(self.dms):
            m.descent_step(self._v(v, k), self._g(g, k), alpha)
        return v

    def descent(self, v, model, b=None, alpha=1e-3, iters=100, g=None, J_hist=None,
                exchange=None):
        """The config-5 loop over the stack: per iteration J, grad J (sub-slab
        interfaces summed, then the rank exchange), v_free -= alpha g."""
        if g is None:
            g = torch.empty(self.nfree_dofs, dtype=torch.float64, device=self.device)
        Jv = J_hist.view(-1, 3) if J_hist is not None else None
        for i in range(iters):
            Ji = Jv[i] if Jv is not None else None
            self.exact_gradient(v, model, b, g=g, J=Ji)
            if exchange is not None:
                exchange.reduce(g, Ji)
            self.descent_step(v, g, alpha)
        return v

    def check(self):
        for m in self.dms:
            m.check()

    def launches(self) -> int:
        return sum(m.launches() for m in self.dms) + self._own_launches

    def time_next(self, start, stop):
        """Arm per-sub-slab events around each sub-slab's dominant kernel of
        the next evaluation; ``kernel_ms`` sums them (``start`` / ``stop``
        are recorded around the whole evaluation's kernels)."""
        self._kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                     for _ in self.dms]
        for a, z in self._kev:
            a.record()
            z.record()
        if not hasattr(self, "_pending"):
            self._pending = []

    def kernel_ms(self) -> list:
        """Sum over sub-slabs of the dominant kernel's time, per armed
        evaluation (synchronises)."""
        torch.cuda.synchronize()
        out = [sum(a.elapsed_time(z) for a, z in ev) for ev in getattr(self, "_pending", [])]
        self._pending = []
        return out
