"""Device-resident evaluation contexts (the B200 side of the drop-in boundary).

``DeviceMesh`` owns one ``fm_ctx`` (include/femmin_b200.h): the frozen Mesh +
Patches of the reference (mesh.py:31-53, patches.py:22-34) uploaded once and
re-laid out as node tiles with 80-byte (3D) / 48-byte (2D) element records.  Its methods take and
return CUDA tensors without host copies; the numpy drop-in functions in
``assembly`` / ``gradients`` are thin wrappers that upload ``v``, call these and
copy the result back.
"""

from __future__ import annotations

import ctypes as C
import os
import sys
import threading
import weakref

import numpy as np
import torch

from . import _lib
from ._device import checked, ptr, require_cuda, stream_ptr, to_dev

DEFAULT_EPS = 1e-8  # gradients.py:20

# ---------------------------------------------------------------------------
# device tensors attached to host objects (Mesh / Patches / LinearLoad)

_ATTACHED: dict[int, dict] = {}


def attach(obj, **tensors):
    key = id(obj)
    if key not in _ATTACHED:
        _ATTACHED[key] = {}
        weakref.finalize(obj, _ATTACHED.pop, key, None)
    _ATTACHED[key].update(tensors)


def attached(obj) -> dict | None:
    return _ATTACHED.get(id(obj))


class DeviceMesh:
    """One evaluation context on the current CUDA device.

    Arguments are CUDA tensors in the reference layout: coords (nn, dim) f64,
    conn (ne, dim+1) i64, volumes (ne,) f64, dphi (dim, ne, dim+1) f64,
    nodes_minim (nfree,) i64 ascending, fixed (nn*d,) u8, and the patch CSR
    p_prefix (nfree,) i64 inclusive, p_elems / p_slot (||T||,) i64.
    """

    def __init__(self, *, dim, d, coords, conn, volumes, dphi, nodes_minim, fixed, p_prefix,
                 p_elems, p_slot, tiling=None):
        self._lib = require_cuda()
        self.dim, self.d = int(dim), int(d)
        self.nn, self.ne = int(coords.shape[0]), int(conn.shape[0])
        self.nfree = int(nodes_minim.shape[0])
        desc = _lib.FmMeshDesc(self.dim, self.d, self.nn, self.ne, ptr(coords), ptr(conn),
                               ptr(volumes), ptr(dphi), self.nfree, ptr(nodes_minim), ptr(fixed),
                               ptr(p_prefix), ptr(p_elems), ptr(p_slot), int(p_elems.shape[0]))
        til = None
        if tiling is not None:
            nt, box = tiling
            til = _lib.FmTiling(int(nt), (C.c_int32 * 3)(*[int(b) for b in box]))
        # the build's temporaries come from the CUDA stream-ordered pool: hand
        # torch's cached (unused) blocks back first
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        if os.environ.get("FM_DEBUG_MEM"):
            print(f"[fm mem] torch allocated before the context build "
                  f"{torch.cuda.memory_allocated() / 1e9:.2f} GB", file=sys.stderr)
        h = C.c_void_p()
        _lib.check(self._lib.fm_ctx_create(C.byref(desc), C.byref(til) if til else None,
                                           stream_ptr(), C.byref(h)), "fm_ctx_create")
        self._h = h
        self._fin = weakref.finalize(self, self._lib.fm_ctx_destroy, h)
        st = _lib.FmCtxStats()
        _lib.check(self._lib.fm_ctx_stats_get(h, C.byref(st)))
        self.stats = {k: getattr(st, k) for k, _ in _lib.FmCtxStats._fields_}
        self.nodes_minim = nodes_minim
        self.nfree_dofs = self._count_free_dofs(fixed, nodes_minim)
        self.device = torch.cuda.current_device()
        self._J = torch.empty(3, dtype=torch.float64, device="cuda")
        # the context's scratch (exchange buffer, partials, status latch) is
        # shared by its launches: the numpy drop-in holds this lock around
        # each call so concurrent callers behave like the pure reference
        # functions
        self.lock = threading.RLock()

    # argument checks: raw pointers go to the kernels, so sizes / dtypes /
    # devices are validated here (ValueError), never by assert
    def _field(self, t, name):
        return checked(t, name, self.nn * self.d, device=self.device)

    def _free(self, t, name):
        return checked(t, name, self.nfree_dofs, device=self.device)

    def _jout(self, t, name="J"):
        return checked(t, name, 3, at_least=True, device=self.device)

    def _count_free_dofs(self, fixed, nodes_minim):
        return int(fixed.numel() - int(fixed.sum().item()))

    def close(self):
        self._fin()

    # ---- evaluation (asynchronous on the current stream) --------------------
    def energy(self, v, model, b=None, densities=None, out=None):
        """J (device double[3]: J, sum vol*W, b.v) of assembly.py:94-106."""
        out = self._J if out is None else self._jout(out, "out")
        self._field(v, "v")
        self._field(b, "b")
        checked(densities, "densities", self.ne, device=self.device)
        m = _model(model)
        _lib.check(self._lib.fm_energy(self._h, C.byref(m), ptr(v), ptr(b), ptr(out),
                                       ptr(densities), stream_ptr()), "fm_energy")
        return out

    def exact_gradient(self, v, model, b=None, g=None, J=None):
        """gradients.py:124-149 into g (nfree_dofs,), fused with J when given."""
        if g is None:
            g = torch.empty(self.nfree_dofs, dtype=torch.float64, device="cuda")
        self._field(v, "v")
        self._field(b, "b")
        self._free(g, "g")
        self._jout(J)
        m = _model(model)
        _lib.check(self._lib.fm_grad_exact(self._h, C.byref(m), ptr(v), ptr(b), ptr(g), ptr(J),
                                           stream_ptr()), "fm_grad_exact")
        return g

    def hvp(self, v, p, model, out=None):
        """Exact Hessian-vector product on the free dofs: d(grad J)(v)[p]
        (fm_hvp_exact).  p: full field (d*nn,), zero on the Dirichlet dofs."""
        if out is None:
            out = torch.empty(self.nfree_dofs, dtype=torch.float64, device="cuda")
        self._field(v, "v")
        self._field(p, "p")
        self._free(out, "out")
        m = _model(model)
        _lib.check(self._lib.fm_hvp_exact(self._h, C.byref(m), ptr(v), ptr(p), ptr(out),
                                          stream_ptr()), "fm_hvp_exact")
        return out

    def numeric_gradient(self, v, model, b=None, eps=DEFAULT_EPS, g=None):
        """gradients.py:84-121 into g (nfree_dofs,)."""
        if g is None:
            g = torch.empty(self.nfree_dofs, dtype=torch.float64, device="cuda")
        self._field(v, "v")
        self._field(b, "b")
        self._free(g, "g")
        m = _model(model)
        _lib.check(self._lib.fm_grad_fd(self._h, C.byref(m), ptr(v), ptr(b), float(eps), ptr(g),
                                        stream_ptr()), "fm_grad_fd")
        return g

    def descent_step(self, v, g, alpha):
        """v_free <- v_free - alpha * g (Dirichlet dofs untouched)."""
        self._field(v, "v")
        self._free(g, "g")
        _lib.check(self._lib.fm_descent_step(self._h, ptr(v), ptr(g), float(alpha),
                                             stream_ptr()))
        return v

    def descent(self, v, model, b=None, alpha=1e-3, iters=100, g=None, J_hist=None,
                exchange=None):
        """Config-5 first-order loop, in place on v: ``iters`` times
        J_hist[i] = J(v), g = grad J(v), v_free -= alpha * g (Dirichlet dofs
        untouched).  J_hist (iters, 3) device doubles or None.  With a
        ``parallel.SlabExchange`` the interface partials of g and J are summed
        across ranks before each update (identical g on both sides of a plane,
        so the shared interface values stay identical)."""
        if g is None:
            g = torch.empty(self.nfree_dofs, dtype=torch.float64, device="cuda")
        self._field(v, "v")
        self._field(b, "b")
        self._free(g, "g")
        if J_hist is not None:
            checked(J_hist, "J_hist", 3 * int(iters), at_least=True, device=self.device)
        if exchange is None:
            m = _model(model)
            _lib.check(self._lib.fm_descent(self._h, C.byref(m), ptr(v), ptr(b), float(alpha),
                                            int(iters), ptr(g), ptr(J_hist), stream_ptr()),
                       "fm_descent")
            return v
        Jv = J_hist.view(-1, 3) if J_hist is not None else None
        for i in range(iters):
            Ji = Jv[i] if Jv is not None else None
            self.exact_gradient(v, model, b, g=g, J=Ji)
            exchange.reduce(g, Ji)
            self.descent_step(v, g, alpha)
        return v

    def check(self):
        """Synchronise and raise InadmissibleStateError for latched conditions."""
        idx = C.c_int64(-1)
        _lib.check(self._lib.fm_ctx_check(self._h, stream_ptr(), C.byref(idx)))

    def launches(self) -> int:
        return int(self._lib.fm_ctx_launches(self._h))

    def time_next(self, start: "torch.cuda.Event", stop: "torch.cuda.Event"):
        """Record the two (already created) CUDA events around the next
        dominant kernel launch of this context."""
        _lib.check(self._lib.fm_ctx_time_next(self._h, C.c_void_p(start.cuda_event),
                                              C.c_void_p(stop.cuda_event)))

    # ---- construction from host objects --------------------------------------
    @classmethod
    def from_host(cls, mesh, patches=None, d=None, tiling=None) -> "DeviceMesh":
        """Upload a (reference-compatible) Mesh + Patches; reuse device copies
        attached by this package's generators."""
        dev = attached(mesh) or {}
        d = int(mesh.d if d is None else d)
        dim = int(mesh.dim)
        coords = dev.get("coords")
        if coords is None:
            coords = to_dev(np.asarray(mesh.nodes2coord, dtype=np.float64))
        conn = dev.get("conn")
        if conn is None:
            conn = to_dev(np.asarray(mesh.elems2nodes, dtype=np.int64))
        vol = dev.get("volumes")
        if vol is None:
            vol = to_dev(np.asarray(mesh.volumes, dtype=np.float64))
        dphi = dev.get("dphi")
        if dphi is None:
            dphi = to_dev(np.stack([np.asarray(g, dtype=np.float64) for g in mesh.dphi]))
        if d == int(mesh.d):
            nm = dev.get("nodes_minim")
            if nm is None:
                nm = to_dev(np.asarray(mesh.nodes_minim, dtype=np.int64))
            fixed = dev.get("fixed")
            if fixed is None:
                fx = np.zeros(mesh.nn * d, dtype=np.uint8)
                fx[np.asarray(mesh.dofs_dirichlet, dtype=np.int64)] = 1
                fixed = to_dev(fx)
        else:  # component count differs from the partition: treat every dof as free
            nm = torch.arange(mesh.nn, dtype=torch.int64, device="cuda")
            fixed = torch.zeros(mesh.nn * d, dtype=torch.uint8, device="cuda")
            patches = None
        if patches is not None:
            pdev = attached(patches) or {}
            prefix = pdev.get("prefix")
            if prefix is None:
                prefix = to_dev(np.asarray(patches.prefix, dtype=np.int64))
            elems = pdev.get("elems")
            if elems is None:
                elems = to_dev(np.asarray(patches.elems, dtype=np.int64))
            slot = pdev.get("slot")
            if slot is None:
                s = getattr(patches, "slot", None)
                if s is None:
                    s = np.argmax(np.asarray(patches.logical), axis=1)
                slot = to_dev(np.asarray(s, dtype=np.int64))
        else:
            from .patches import build_patches_device
            prefix, elems, slot = build_patches_device(conn, nm, mesh.nn, dim + 1)
        return cls(dim=dim, d=d, coords=coords, conn=conn, volumes=vol, dphi=dphi,
                   nodes_minim=nm, fixed=fixed, p_prefix=prefix, p_elems=elems, p_slot=slot,
                   tiling=tiling)


def _model(model) -> _lib.FmModel:
    if isinstance(model, _lib.FmModel):
        return model
    from .models import fm_model_struct
    return fm_model_struct(model)


# ---------------------------------------------------------------------------
# context cache for the numpy drop-in (frozen Mesh / Patches are immutable)
#
# One context per (mesh, d): build_patches is a deterministic function of the
# mesh (patches.py:37-71), so the energy call (no patches) and the gradient
# calls (the user's Patches) share it.  A Patches object is checked once
# against the canonical CSR built on the device; only a non-canonical one
# (a hand-made patch structure) gets a context of its own.

_CTX: dict[tuple, DeviceMesh] = {}
_CANONICAL: dict[tuple, set] = {}  # (id(mesh), d) -> ids of Patches equal to the canonical CSR


def _drop(key):
    ctx = _CTX.pop(key, None)
    if ctx is not None:
        ctx.close()
    _CANONICAL.pop(key, None)


def _patch_arrays(patches):
    pdev = attached(patches) or {}
    prefix = pdev.get("prefix")
    if prefix is None:
        prefix = to_dev(np.asarray(patches.prefix, dtype=np.int64))
    elems = pdev.get("elems")
    if elems is None:
        elems = to_dev(np.asarray(patches.elems, dtype=np.int64))
    slot = pdev.get("slot")
    if slot is None:
        s = getattr(patches, "slot", None)
        if s is None:
            s = np.argmax(np.asarray(patches.logical), axis=1)
        slot = to_dev(np.asarray(s, dtype=np.int64))
    return prefix, elems, slot


def _is_canonical(mesh, patches, d) -> bool:
    if d != int(mesh.d):
        return True  # the patches are not used (every dof free)
    from .patches import build_patches_device
    dev = attached(mesh) or {}
    conn = dev.get("conn")
    if conn is None:
        conn = to_dev(np.asarray(mesh.elems2nodes, dtype=np.int64))
    nm = dev.get("nodes_minim")
    if nm is None:
        nm = to_dev(np.asarray(mesh.nodes_minim, dtype=np.int64))
    ref = build_patches_device(conn, nm, int(mesh.nn), int(mesh.dim) + 1)
    got = _patch_arrays(patches)
    return all(a.shape == b.shape and bool(torch.equal(a, b)) for a, b in zip(ref, got))


_CTX_LOCK = threading.RLock()


def context_for(mesh, patches=None, d=None) -> DeviceMesh:
    with _CTX_LOCK:
        return _context_for(mesh, patches, d)


def _context_for(mesh, patches=None, d=None) -> DeviceMesh:
    d = int(mesh.d if d is None else d)
    key = (id(mesh), d)
    if patches is not None:
        seen = _CANONICAL.get(key)
        if seen is None or id(patches) not in seen:
            if not _is_canonical(mesh, patches, d):
                key = (id(mesh), id(patches), d)
            else:
                _CANONICAL.setdefault(key, set()).add(id(patches))
                weakref.finalize(patches, lambda k=key, i=id(patches):
                                 _CANONICAL.get(k, set()).discard(i))
    ctx = _CTX.get(key)
    if ctx is None:
        ctx = DeviceMesh.from_host(mesh, patches if len(key) == 3 else None, d)
        _CTX[key] = ctx
        weakref.finalize(mesh, _drop, key)
        if len(key) == 3:
            weakref.finalize(patches, _drop, key)
    return ctx
