"""Density models: the plugin surface of models.py (reference) on the GPU.

Same classes, names, validation and exceptions as
``/root/reference/pkg/src/femmin/models.py``; the batched functions evaluate
on the device through ``fm_density_rows`` / ``fm_det_rows`` (fp64, reference
operation order, see csrc/fm_density.cuh).  Inputs and outputs are nested
lists ``F[j][m]`` of equally sized numpy arrays, as in the reference.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._device import ptr, require_cuda, stream_ptr, to_dev, to_host


class InadmissibleStateError(ValueError):
    """det F <= 0 where the exact derivative formulas are meaningless (models.py:16-17)."""


@dataclass(frozen=True)
class ElasticParams:
    """Young's modulus / Poisson ratio with derived constants (models.py:20-47)."""

    E: float
    nu: float

    def __post_init__(self):
        if self.E <= 0:
            raise ValueError("Young's modulus must be positive")
        if not 0.0 < self.nu < 0.5:
            raise ValueError("Poisson ratio must lie in (0, 0.5)")

    @property
    def mu(self) -> float:
        return self.E / (2.0 * (1.0 + self.nu))

    @property
    def bulk(self) -> float:
        return self.E / (3.0 * (1.0 - 2.0 * self.nu))

    @property
    def C1(self) -> float:
        return self.mu / 2.0

    @property
    def D1(self) -> float:
        return self.bulk / 2.0


@dataclass(frozen=True)
class LameParams:
    """Direct (C1, D1) constants.  The benchmark configs use D1 = lambda/2
    (SURVEY §0.1 #1); the kernels read only C1 and D1 (models.py:97, 112-117)."""

    C1: float
    D1: float

    @classmethod
    def from_young_poisson(cls, E: float, nu: float) -> "LameParams":
        mu = E / (2.0 * (1.0 + nu))
        lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
        return cls(mu / 2.0, lam / 2.0)


@dataclass(frozen=True)
class PLaplaceParams:
    p: float

    def __post_init__(self):
        if self.p <= 1.0:
            raise ValueError("p-Laplacian exponent must satisfy p > 1")


# the densities the CUDA engine implements: this package's classes and the
# reference's own (femmin.models), matched by exact type
_ENGINE_MODELS = {
    ("paper_2109_01158_b200.models", "NeoHookean"): _lib.FM_MODEL_NEOHOOKEAN,
    ("femmin.models", "NeoHookean"): _lib.FM_MODEL_NEOHOOKEAN,
    ("paper_2109_01158_b200.models", "PLaplacian"): _lib.FM_MODEL_PLAPLACE,
    ("femmin.models", "PLaplacian"): _lib.FM_MODEL_PLAPLACE,
}


def fm_model_struct(model) -> _lib.FmModel:
    """C view of a model plugin (models.py:141-170: .d .dim .params).

    The GPU kernels evaluate the Neo-Hookean and p-Laplace densities
    themselves, so only models whose density IS one of those are accepted:
    instances of exactly this package's or the reference's NeoHookean /
    PLaplacian with their own density / ddensity.  A subclass, a duck-typed
    plugin or an instance with an overridden density would otherwise get the
    built-in law silently; it raises NotImplementedError instead (there is no
    CPU fallback).
    """
    cls = type(model)
    kind = _ENGINE_MODELS.get((cls.__module__, cls.__qualname__))
    if kind is None:
        raise NotImplementedError(
            f"{cls.__module__}.{cls.__qualname__}: the GPU engine evaluates the built-in "
            "NeoHookean and PLaplacian densities only (models.py:141-170); custom density "
            "plugins are not supported")
    for name in ("density", "ddensity"):
        if name in getattr(model, "__dict__", {}):
            raise NotImplementedError(
                f"model.{name} is overridden on the instance; the GPU engine evaluates the "
                "built-in density only")
    prm = model.params
    if kind == _lib.FM_MODEL_PLAPLACE:
        if int(model.d) != 1:
            raise ValueError("p-Laplacian model must have d = 1")
        return _lib.FmModel(kind, int(model.dim), float(prm.p), 0.0, 0.0)
    return _lib.FmModel(kind, int(model.dim), 0.0, float(prm.C1), float(prm.D1))


def _stack(F):
    rows = np.asarray(F[0][0]).shape
    flat = np.stack([np.asarray(F[j][m], dtype=np.float64).reshape(-1)
                     for j in range(len(F)) for m in range(len(F[0]))])
    return flat, rows


def _unstack(flat, rows, D, dim):
    return [[flat[j * dim + m].reshape(rows) for m in range(dim)] for j in range(D)]


def _rows_call(model_struct, F, want_W: bool, want_P: bool):
    lib = require_cuda()
    flat, rows = _stack(F)
    D, dim = len(F), len(F[0])
    n = flat.shape[1]
    Fd = to_dev(flat)
    W = torch.empty(n, dtype=torch.float64, device="cuda") if want_W else None
    P = torch.empty_like(Fd) if want_P else None
    nbad = C.c_int64(0)
    _lib.check(lib.fm_density_rows(C.byref(model_struct), n, ptr(Fd), ptr(W), ptr(P),
                                   C.byref(nbad), stream_ptr()))
    Wh = to_host(W).reshape(rows) if want_W else None
    Ph = _unstack(to_host(P), rows, D, dim) if want_P else None
    return Wh, Ph, int(nbad.value)


def batch_determinant(F):
    """models.py:59-71."""
    lib = require_cuda()
    flat, rows = _stack(F)
    Fd = to_dev(flat)
    det = torch.empty(flat.shape[1], dtype=torch.float64, device="cuda")
    _lib.check(lib.fm_det_rows(len(F), flat.shape[1], ptr(Fd), ptr(det), None, stream_ptr()))
    return to_host(det).reshape(rows)


def batch_cofactor(F):
    """models.py:74-86."""
    lib = require_cuda()
    flat, rows = _stack(F)
    Fd = to_dev(flat)
    cof = torch.empty_like(Fd)
    _lib.check(lib.fm_det_rows(len(F), flat.shape[1], ptr(Fd), None, ptr(cof), stream_ptr()))
    return _unstack(to_host(cof), rows, len(F), len(F))


def _nh_struct(params, dim):
    return _lib.FmModel(_lib.FM_MODEL_NEOHOOKEAN, dim, 0.0, float(params.C1), float(params.D1))


def neo_hookean_density(F, params) -> np.ndarray:
    """models.py:89-100 (+inf where det F <= 0)."""
    return _rows_call(_nh_struct(params, len(F)), F, True, False)[0]


def neo_hookean_ddensity(F, params):
    """models.py:103-120; raises InadmissibleStateError if any det F <= 0."""
    _, P, nbad = _rows_call(_nh_struct(params, len(F)), F, False, True)
    if nbad:
        raise InadmissibleStateError("nonpositive det F in the exact derivative path")
    return P


def _pl_struct(params, dim):
    return _lib.FmModel(_lib.FM_MODEL_PLAPLACE, dim, float(params.p), 0.0, 0.0)


def p_laplacian_density(G, params) -> np.ndarray:
    """models.py:123-126."""
    return _rows_call(_pl_struct(params, len(G[0])), G, True, False)[0]


def p_laplacian_ddensity(G, params):
    """models.py:129-138."""
    return _rows_call(_pl_struct(params, len(G[0])), G, False, True)[1]


class NeoHookean:
    """Vector density model: d = dim components (models.py:141-155)."""

    def __init__(self, params, dim: int):
        if dim not in (2, 3):
            raise ValueError("Neo-Hookean model needs dim in {2, 3}")
        self.params = params
        self.dim = dim
        self.d = dim

    def density(self, F):
        return neo_hookean_density(F, self.params)

    def ddensity(self, F):
        return neo_hookean_ddensity(F, self.params)


class PLaplacian:
    """Scalar density model (d = 1) for any spatial dimension (models.py:158-170)."""

    def __init__(self, params: PLaplaceParams, dim: int):
        self.params = params
        self.dim = dim
        self.d = 1

    def density(self, G):
        return p_laplacian_density(G, self.params)

    def ddensity(self, G):
        return p_laplacian_ddensity(G, self.params)
