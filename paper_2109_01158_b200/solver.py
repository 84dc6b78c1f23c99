"""Minimizers over the free dofs with the Dirichlet values held fixed
(the main consumer of J / grad J; reference solver.py).

The same two methods and options as the reference:

* ``"tr"`` — Hessian-free trust-region Newton (solver.py:179-231): the model
  step by Steihaug truncated CG (solver.py:77-113) with Hessian-vector
  products from central differences of the gradient (solver.py:64-74), forcing
  term eta = min(1/2, sqrt(|g| / |g0|_inf)), ratio test 1/4 - 3/4;
* ``"lbfgs"`` — L-BFGS with Armijo backtracking that rejects +inf trials
  (solver.py:234-283, two-loop recursion 286-300);

plus ``continuation_solve`` (warm-started load stepping, solver.py:303-331).

Here every vector of the iteration (iterate, gradient, CG directions, L-BFGS
pairs) is a torch tensor.  ``minimize_device`` keeps them on the GPU and calls
the device engine (``DeviceMesh``: energy-only kernel for trial points, the
fused exact-gradient kernel without J for gradients and Hessian-vector
products), so a CG iteration costs two gradient launches and two scalar reads,
with no host copies of fields.  ``minimize`` is the reference's signature
(host callables J(v) -> float, g(v) -> free-dof gradient on numpy fields) on
CPU tensors.
"""

from __future__ import annotations

import math
import sys
import time
from dataclasses import dataclass

import numpy as np
import torch


class InvalidStartError(ValueError):
    """The initial field has non-finite energy (solver.py:21-22)."""


class StagnationError(RuntimeError):
    """No admissible step at the minimal trust radius (solver.py:25-26)."""


@dataclass
class SolveOptions:
    """solver.py:29-47 (same fields, defaults and validation)."""
    solver: str = "tr"
    tol_g: float = 1e-6
    tol_step: float = 1e-6
    tol_f: float = 1e-6
    max_iters: int = 2000
    tr_radius0: float = 1.0
    tr_radius_max: float = 1e10
    max_cg: int | None = None
    hvp_step: float | None = None  # None: sqrt(eps_mach) (1 + |x|) / |dir|
    lbfgs_memory: int = 10
    verbose: bool = False
    # new (not in the reference): "exact" makes minimize_device's trust-region
    # CG use the engine's exact Hessian-vector product (fm_hvp_exact, one
    # launch) instead of central differences of two gradients
    hvp: str = "fd"
    # new: minimize_device runs the trust region's CG on the device
    # (csrc/fm_cg.cu, one flag read per CG iteration); False: the host loop
    device_cg: bool = True

    def __post_init__(self):
        if min(self.tol_g, self.tol_step, self.tol_f) <= 0:
            raise ValueError("tolerances must be positive")
        if self.solver not in ("tr", "lbfgs"):
            raise ValueError(f"unknown solver {self.solver!r}")
        if self.hvp not in ("fd", "exact"):
            raise ValueError(f"unknown Hessian-vector product {self.hvp!r}")


@dataclass
class MinimizeResult:
    """solver.py:50-61.  ``u`` is the full field (Dirichlet entries exactly
    as given): a numpy array from ``minimize``, a CUDA tensor from
    ``minimize_device``."""
    u: object
    J_u: float
    iters: int
    grad_norm: float
    time: float
    converged: bool
    status: str
    J_grad_u: float | None = None
    n_energy: int = 0
    n_grad: int = 0


_SQRT_EPS = math.sqrt(np.finfo(float).eps)


def _dot(a, b) -> float:
    return float(torch.dot(a, b))


def _nrm(a) -> float:
    return float(torch.linalg.vector_norm(a))


def _nrm_inf(a) -> float:
    return float(a.abs().max()) if a.numel() else 0.0


def _steihaug(g, hvp, radius, rtol, maxiter):
    """Truncated CG for min g.z + z.Hz/2, |z| <= radius: (z, hit_boundary)."""
    z = torch.zeros_like(g)
    r = -g
    d = r.clone()
    rr = _dot(r, r)
    if math.sqrt(rr) <= rtol:
        return z, False

    def boundary(z, d):
        dd, zd, zz = _dot(d, d), _dot(z, d), _dot(z, z)
        tau = (-zd + math.sqrt(zd * zd + dd * (radius * radius - zz))) / dd
        return z + tau * d

    for _ in range(maxiter):
        Hd = hvp(d)
        dHd = _dot(d, Hd)
        if dHd <= 0.0:
            return boundary(z, d), True
        alpha = rr / dHd
        z_new = z + alpha * d
        if _nrm(z_new) >= radius:
            return boundary(z, d), True
        z = z_new
        r = r - alpha * Hd
        rr_new = _dot(r, r)
        if math.sqrt(rr_new) <= rtol:
            return z, False
        d = r + (rr_new / rr) * d
        rr = rr_new
    return z, False


def _trust_region(fx, gx, x, f, opts, hx=None, cg=None):
    g = gx(x)
    gn0 = _nrm_inf(g)
    gtol = opts.tol_g * max(1.0, gn0)
    radius = opts.tr_radius0
    max_cg = opts.max_cg or max(2 * x.numel(), 10)
    status, converged, it = "max-iters", False, 0
    for it in range(1, opts.max_iters + 1):
        gn = _nrm_inf(g)
        if gn <= gtol:
            status, converged = "gradient-tolerance", True
            break
        if opts.verbose:
            print(f"tr iter {it:4d}  J={f: .8e}  |g|={gn:.3e}  radius={radius:.3e}",
                  file=sys.stderr)
        xnorm = _nrm(x)

        def hvp(p):
            if hx is not None:  # exact product at x (admissible: f(x) is finite)
                return hx(x, p)
            pn = _nrm(p)
            if pn == 0.0:
                return torch.zeros_like(p)
            h = opts.hvp_step or _SQRT_EPS * (1.0 + xnorm) / pn
            return (gx(x + h * p) - gx(x - h * p)) / (2.0 * h)

        g2 = _nrm(g)
        eta = min(0.5, math.sqrt(g2 / max(gn0, 1e-300)))
        if cg is not None:  # device-resident CG: scalars and decisions on the GPU
            p, _ = cg.solve(g, x, xnorm, radius, eta * g2, max_cg, opts.hvp_step)
        else:
            p, _ = _steihaug(g, hvp, radius, eta * g2, max_cg)
        pred = -(_dot(g, p) + 0.5 * _dot(p, hvp(p)))
        pn = _nrm(p)
        if pred <= 0.0 or pn == 0.0:
            radius *= 0.25
            if radius < 1e-14 * (1.0 + xnorm):
                raise StagnationError(f"no model decrease at radius {radius:.3e}, |g|={gn:.3e}")
            continue
        f_trial = fx(x + p)
        ratio = (f - f_trial) / pred if math.isfinite(f_trial) else 0.0
        if ratio < 0.25:
            radius = 0.25 * min(radius, pn)
        elif ratio > 0.75 and pn >= 0.99 * radius:
            radius = min(2.0 * radius, opts.tr_radius_max)
        if ratio > 1e-4 and f_trial < f:
            x = x + p
            f_prev, f = f, f_trial
            g = gx(x)
            if (pn <= opts.tol_step * (1.0 + _nrm(x))
                    and (f_prev - f) <= opts.tol_f * (1.0 + abs(f))):
                status, converged = "step-tolerance", True
                break
        elif radius < 1e-14 * (1.0 + xnorm):
            raise StagnationError(f"trial steps rejected down to radius {radius:.3e}")
    return x, f, it, _nrm_inf(g), converged, status


def _lbfgs_direction(g, S, Y):
    q = -g
    if not S:
        return q
    rhos = [1.0 / _dot(y, s) for s, y in zip(S, Y)]
    alphas = []
    for s, y, rho in zip(reversed(S), reversed(Y), reversed(rhos)):
        a = rho * _dot(s, q)
        alphas.append(a)
        q = q - a * y
    q = q * (_dot(S[-1], Y[-1]) / _dot(Y[-1], Y[-1]))
    for (s, y, rho), a in zip(zip(S, Y, rhos), reversed(alphas)):
        q = q + (a - rho * _dot(y, q)) * s
    return q


def _lbfgs(fx, gx, x, f, opts):
    S, Y = [], []
    g = gx(x)
    gtol = opts.tol_g * max(1.0, _nrm_inf(g))
    status, converged, it = "max-iters", False, 0
    for it in range(1, opts.max_iters + 1):
        gn = _nrm_inf(g)
        if gn <= gtol:
            status, converged = "gradient-tolerance", True
            break
        if opts.verbose:
            print(f"lbfgs iter {it:4d}  J={f: .8e}  |g|={gn:.3e}", file=sys.stderr)
        d = _lbfgs_direction(g, S, Y)
        gd = _dot(g, d)
        if gd >= 0.0:
            d = -g
            gd = _dot(g, d)
        step, ok = 1.0, False
        for _ in range(60):
            f_trial = fx(x + step * d)
            if math.isfinite(f_trial) and f_trial <= f + 1e-4 * step * gd:
                ok = True
                break
            step *= 0.5
        if not ok:
            raise StagnationError("line search failed at minimal step")
        x_new = x + step * d
        g_new = gx(x_new)
        s, y = x_new - x, g_new - g
        if _dot(s, y) > 1e-12 * _dot(s, s):
            S.append(s)
            Y.append(y)
            if len(S) > opts.lbfgs_memory:
                S.pop(0)
                Y.pop(0)
        f_prev, f = f, float(f_trial)
        x, g = x_new, g_new
        if (_nrm(s) <= opts.tol_step * (1.0 + _nrm(x))
                and (f_prev - f) <= opts.tol_f * (1.0 + abs(f))):
            status, converged = "step-tolerance", True
            break
    return x, f, it, _nrm_inf(g), converged, status


def _run(fx, gx, x0, opts, hx=None, cg=None):
    f0 = fx(x0)
    if not math.isfinite(f0):
        raise InvalidStartError("initial field has non-finite energy")
    if opts.solver == "lbfgs":
        return _lbfgs(fx, gx, x0, f0, opts)
    return _trust_region(fx, gx, x0, f0, opts, hx, cg)


class _DeviceSteihaug:
    """Steihaug truncated CG (solver.py:77-113) with every vector and scalar
    on the device (csrc/fm_cg.cu): per iteration the Hessian-vector product
    (two gradient launches around x -/+ h d, or one exact-HVP launch), three
    fused vector kernels that also decide alpha / beta / boundary / tolerance,
    and ONE 24-byte read of the done flags; the host never waits on a CG
    scalar.  Same iterates as _steihaug up to the summation order of the dot
    products."""

    def __init__(self, dm, model, b, work, count, exact, embed):
        from . import _lib
        self.lib = _lib.load()
        self._lib = _lib
        self.dm, self.model, self.b, self.work, self.count = dm, model, b, work, count
        self.exact, self.embed = exact, embed
        n = dm.nfree_dofs
        f64 = dict(dtype=torch.float64, device=work.device)
        self.z, self.znew, self.r, self.d, self.Hd = (torch.empty(n, **f64) for _ in range(5))
        self.gp, self.gm = torch.empty(n, **f64), torch.empty(n, **f64)
        self.st = torch.zeros(32, **f64)
        self.part = torch.empty(self.lib.fm_cg_scratch_doubles(), **f64)
        self.ticket = torch.zeros(1, dtype=torch.int32, device=work.device)
        self.flags = torch.empty(3, dtype=torch.float64, pin_memory=True)
        self.pfull = torch.zeros_like(work) if exact else None
        self.n = n

    def _p(self, t):
        return None if t is None else t.data_ptr()

    def solve(self, g, x, xnorm, radius, rtol, maxiter, hvp_step=None):
        from ._device import stream_ptr
        lib, P, s = self.lib, self._p, stream_ptr()
        init = torch.zeros(32, dtype=torch.float64)
        init[4], init[5] = radius, rtol
        init[13] = _SQRT_EPS * (1.0 + xnorm)
        init[18] = hvp_step or 0.0
        self.st.copy_(init)
        chk = self._lib.check
        chk(lib.fm_cg_init(self.n, P(g), P(self.r), P(self.d), P(self.z), P(self.st),
                           P(self.part), P(self.ticket), s))
        if not self._done():
            work = self.work
            if self.exact:
                xf = self.embed(x)  # the field is fixed during one CG solve
            for _ in range(maxiter):
                if self.exact:
                    chk(lib.fm_cg_embed(self.dm._h, None, P(self.d), P(self.st), 0, 1.0,
                                        P(self.pfull), s))
                    self.dm.hvp(xf, self.pfull, self.model, out=self.Hd)
                    self.count["h"] = self.count.get("h", 0) + 1
                    gp = gm = None
                else:
                    for sign, out in ((1.0, self.gp), (-1.0, self.gm)):
                        chk(lib.fm_cg_embed(self.dm._h, P(x), P(self.d), P(self.st), 1, sign,
                                            P(work), s))
                        self.dm.exact_gradient(work, self.model, self.b, g=out)
                    self.count["g"] += 2
                    gp, gm = self.gp, self.gm
                chk(lib.fm_cg_iterate(self.n, P(gp), P(gm), P(self.Hd), P(self.z),
                                      P(self.znew), P(self.r), P(self.d), P(self.st),
                                      P(self.part), P(self.ticket), s))
                if self._done():
                    break
        return self.z.clone(), bool(self.flags[1] != 0.0)

    def _done(self) -> bool:
        # one small read per iteration; dm.check() synchronises the stream and
        # raises for an inadmissible gradient / product (models.py:107-110)
        self.flags.copy_(self.st[16:19], non_blocking=True)
        self.dm.check()
        return bool(self.flags[0] != 0.0)


def minimize(J, g, v0, dofs_minim, opts: SolveOptions | None = None) -> MinimizeResult:
    """The reference signature (solver.py:116-176): J maps a full numpy field
    to a float (+inf when inadmissible), g to the free-dof gradient; the
    Dirichlet entries of v0 are preserved bit-exactly."""
    opts = opts or SolveOptions()
    template = np.array(v0, dtype=float, copy=True)
    dofs = np.asarray(dofs_minim, dtype=np.int64)
    count = {"f": 0, "g": 0}

    def embed(x):
        v = template.copy()
        v[dofs] = x.numpy()
        return v

    def fx(x):
        count["f"] += 1
        return float(J(embed(x)))

    def gx(x):
        count["g"] += 1
        return torch.from_numpy(np.ascontiguousarray(g(embed(x)), dtype=float))

    t0 = time.perf_counter()
    x, f, it, gn, conv, status = _run(fx, gx, torch.from_numpy(template[dofs].copy()), opts)
    return MinimizeResult(u=embed(x), J_u=f, iters=it, grad_norm=gn,
                          time=time.perf_counter() - t0, converged=conv, status=status,
                          n_energy=count["f"], n_grad=count["g"])


def minimize_device(dm, model, b, v0: torch.Tensor, dofs_minim: torch.Tensor,
                    opts: SolveOptions | None = None) -> MinimizeResult:
    """Device-resident minimization of J(v) = sum |T| W(grad v) - b.v over the
    free dofs of ``v0`` (a CUDA tensor, full interleaved field) with the
    engine of ``dm`` (a ``DeviceMesh``).  ``dofs_minim``: free dof indices
    (CUDA int64, ascending).  Trial energies use the energy kernel, gradients
    the exact-gradient kernel; inadmissible gradients raise
    InadmissibleStateError as the reference's g does (models.py:107-110)."""
    opts = opts or SolveOptions()
    template = v0.detach().to(torch.float64).clone()
    dofs = dofs_minim.to(device=template.device, dtype=torch.int64)
    J3 = torch.empty(3, dtype=torch.float64, device=template.device)
    work = template.clone()  # full field the kernels read; only free dofs are rewritten
    count = {"f": 0, "g": 0}

    def embed(x):
        return work.index_copy_(0, dofs, x)

    def fx(x):
        count["f"] += 1
        return float(dm.energy(embed(x), model, b, out=J3)[0])

    def gx(x):
        count["g"] += 1
        gr = dm.exact_gradient(embed(x), model, b)
        dm.check()
        return gr

    hx = None
    if opts.hvp == "exact":
        pfull = torch.zeros_like(template)  # direction, zero on the Dirichlet dofs

        def hx(x, p):
            count["h"] = count.get("h", 0) + 1
            return dm.hvp(embed(x), pfull.index_copy_(0, dofs, p), model)

    cg = None
    if opts.solver == "tr" and opts.device_cg:
        cg = _DeviceSteihaug(dm, model, b, work, count, opts.hvp == "exact", embed)
    t0 = time.perf_counter()
    x, f, it, gn, conv, status = _run(fx, gx, template.index_select(0, dofs), opts, hx, cg)
    torch.cuda.synchronize()
    res = MinimizeResult(u=template.index_copy(0, dofs, x), J_u=f, iters=it, grad_norm=gn,
                         time=time.perf_counter() - t0, converged=conv, status=status,
                         n_energy=count["f"], n_grad=count["g"])
    res.n_hvp = count.get("h", 0)
    return res


def continuation_solve(J, g, v0, dofs_minim, dofs_dirichlet, dirichlet_values,
                       opts: SolveOptions | None = None, callback=None):
    """Warm-started load stepping (solver.py:303-331): step t overwrites the
    Dirichlet entries with dirichlet_values[t - 1] and starts from the
    previous minimizer; errors are annotated with the load step."""
    results = []
    v = np.array(v0, dtype=float, copy=True)
    for t, bc in enumerate(dirichlet_values, start=1):
        v[dofs_dirichlet] = bc
        try:
            res = minimize(J, g, v, dofs_minim, opts)
        except (InvalidStartError, StagnationError) as exc:
            raise type(exc)(f"load step {t}: {exc}") from exc
        results.append(res)
        v = np.array(res.u, dtype=float, copy=True)
        if callback is not None:
            callback(t, res)
    return results
