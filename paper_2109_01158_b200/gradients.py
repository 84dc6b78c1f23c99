"""Exact and nodal-patch FD gradient engines (GPU): mirror of gradients.py.

Both engines run as node-tile kernels over the cached device context
(csrc/fm_eval_exact.cu, csrc/fm_eval_ref.cu): per element F, dW/dF (exact)
or the 2*d perturbed densities per owned slot (FD), staged in shared memory
and summed per free dof in ascending element order, without float atomics.
Outputs follow ``mesh.dofs_minim`` order exactly like ``_blocks_to_dofs``
(gradients.py:68-74); errors are the reference's InadmissibleStateError
messages.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from ._device import to_dev, to_host
from .assembly import LinearLoad, _check_field, _load_device
from .device import DEFAULT_EPS, context_for
from .mesh import Mesh
from .patches import Patches


@dataclass(frozen=True)
class GradientConfig:
    """gradients.py:23-32."""

    mode: str = "numeric"
    eps: float = DEFAULT_EPS

    def __post_init__(self):
        if self.mode not in ("numeric", "exact"):
            raise ValueError(f"unknown gradient mode {self.mode!r}")
        if self.mode == "numeric" and self.eps <= 0:
            raise ValueError("central-difference step must be positive")


def dF_dv_table(patches: Patches):
    """dF[j,m]/dv_n on every patch row: the owner's basis gradient (gradients.py:54-56)."""
    return [np.asarray(dm)[np.asarray(patches.logical)] for dm in patches.dphi]


def _prep(v, mesh, patches, model):
    d = model.d
    if d != mesh.d:
        raise ValueError(f"model has {d} components but the mesh partition has {mesh.d}")
    v = _check_field(v, mesh, d)
    return context_for(mesh, patches, d), to_dev(v)


def exact_gradient(v: np.ndarray, mesh: Mesh, patches: Patches, model,
                   load: LinearLoad | None = None) -> np.ndarray:
    """Chain-rule gradient through dW/dF on the free dofs (gradients.py:124-149)."""
    ctx, vd = _prep(v, mesh, patches, model)
    with ctx.lock:
        g = ctx.exact_gradient(vd, model, _load_device(load))
        ctx.check()
        return to_host(g)


def numeric_gradient(v: np.ndarray, mesh: Mesh, patches: Patches, model,
                     load: LinearLoad | None = None, eps: float = DEFAULT_EPS) -> np.ndarray:
    """Patch-localised central differences, all dofs at once (gradients.py:84-121)."""
    if eps <= 0:
        raise ValueError("central-difference step must be positive")
    ctx, vd = _prep(v, mesh, patches, model)
    with ctx.lock:
        g = ctx.numeric_gradient(vd, model, _load_device(load), eps)
        ctx.check()
        return to_host(g)


def gradient(v, mesh, patches, model, load=None, cfg: GradientConfig | None = None):
    """Dispatch on the configured engine (gradients.py:152-157)."""
    cfg = cfg or GradientConfig()
    if cfg.mode == "exact":
        return exact_gradient(v, mesh, patches, model, load)
    return numeric_gradient(v, mesh, patches, model, load, eps=cfg.eps)


def energy_and_gradient(v, mesh, patches, model, load=None, cfg: GradientConfig | None = None):
    """New, additive: J and the gradient in one call (one fused pass for the
    exact engine).  Returns (J, g); raises like ``gradient``."""
    cfg = cfg or GradientConfig(mode="exact")
    ctx, vd = _prep(v, mesh, patches, model)
    b = _load_device(load)
    J = torch.empty(3, dtype=torch.float64, device="cuda")
    with ctx.lock:
        if cfg.mode == "exact":
            g = ctx.exact_gradient(vd, model, b, J=J)
        else:
            ctx.energy(vd, model, b, out=J)
            g = ctx.numeric_gradient(vd, model, b, cfg.eps)
        ctx.check()
        return float(to_host(J)[0]), to_host(g)
