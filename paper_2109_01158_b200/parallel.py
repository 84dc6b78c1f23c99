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
        self.rank, self.world, self.group = rank, world, group
        nxl = ix1 - ix0
        dev = dofs_minim.device
        self.left = (plane_dof_positions(plane_nodes(0, nxl, ny, nz, dev), d, dofs_minim)
                     if rank > 0 else None)
        self.right = (plane_dof_positions(plane_nodes(nxl, nxl, ny, nz, dev), d, dofs_minim)
                      if rank < world - 1 else None)
        # both planes packed / added back with one launch each: positions
        # [left | right], send and receive buffers with the same layout
        planes = [p for p in (self.left, self.right) if p is not None]
        self.pos = torch.cat(planes) if planes else None
        n = (ny + 1) * (nz + 1) * d
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
