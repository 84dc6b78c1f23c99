"""CPU-side checks of the boundary: the C-ABI library loads and exports every
symbol include/femmin_b200.h declares, the ctypes table matches the header,
and the host-side validation mirrors the reference (no compute calls)."""

import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "femmin_b200.h")


def _declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fm_[A-Za-z0-9_]+)\s*\(", text)))


def test_library_builds_and_exports_every_declared_symbol():
    from paper_2109_01158_b200 import _lib, build
    path = build.build()
    assert os.path.exists(path)
    lib = ctypes.CDLL(path)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert len(_declared()) >= 25


def test_ctypes_table_covers_header():
    from paper_2109_01158_b200 import _lib
    assert set(_declared()) == set(_lib.SIGNATURES), (
        set(_declared()) ^ set(_lib.SIGNATURES))
    lib = _lib.load()
    assert lib.fm_version() == 1


def test_host_validation_without_gpu():
    """Argument errors are reported without touching the device."""
    from paper_2109_01158_b200 import _lib
    lib = _lib.load()
    nn, ne = ctypes.c_int64(), ctypes.c_int64()
    assert lib.fm_lshape_sizes(4, ctypes.byref(nn), ctypes.byref(ne)) == _lib.FM_OK
    assert (nn.value, ne.value) == (3201, 6144)          # cfg1
    assert lib.fm_lshape_sizes(10, ctypes.byref(nn), ctypes.byref(ne)) == _lib.FM_OK
    assert (nn.value, ne.value) == (12591105, 25165824)  # cfg2
    assert lib.fm_lshape_sizes(-1, ctypes.byref(nn), ctypes.byref(ne)) == _lib.FM_INVALID_ARG
    assert "level" in _lib.last_error()
    with pytest.raises(ValueError):
        _lib.check(_lib.FM_INVALID_ARG)


def test_reference_validation_mirrored():
    from paper_2109_01158_b200 import (ElasticParams, GradientConfig, NeoHookean,
                                       PLaplaceParams, PLaplacian)
    with pytest.raises(ValueError):
        ElasticParams(E=-1.0, nu=0.3)
    with pytest.raises(ValueError):
        ElasticParams(E=1.0, nu=0.6)
    with pytest.raises(ValueError):
        PLaplaceParams(p=1.0)
    with pytest.raises(ValueError):
        GradientConfig(mode="autodiff")
    with pytest.raises(ValueError):
        GradientConfig(mode="numeric", eps=0.0)
    assert GradientConfig().mode == "numeric"
    with pytest.raises(ValueError):
        NeoHookean(ElasticParams(E=1.0, nu=0.3), dim=4)
    nh = NeoHookean(ElasticParams(E=1.0, nu=0.3), dim=2)
    assert nh.d == 2 and nh.dim == 2
    pl = PLaplacian(PLaplaceParams(p=3.0), dim=2)
    assert pl.d == 1 and pl.dim == 2
    p = ElasticParams(E=2e8, nu=0.3)
    assert p.mu == pytest.approx(2e8 / 2.6) and p.bulk == pytest.approx(2e8 / 1.2)


def test_product_path_fails_loudly_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    from paper_2109_01158_b200 import _lib, generate_lshape_mesh_2d
    with pytest.raises(_lib.FemminCudaError):
        generate_lshape_mesh_2d(1)


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2109_01158_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                bad = re.findall(r"(from\s+oracle|import\s+oracle|femmin_oracle|oracle/_ref)",
                                 src)
                assert not bad, (f, bad)


def test_model_dispatch_is_strict():
    """Only the built-in densities reach the kernels (a subclass or a
    duck-typed plugin must not silently get the Neo-Hookean / p-Laplace law)."""
    from paper_2109_01158_b200 import (ElasticParams, NeoHookean, PLaplaceParams,
                                       PLaplacian, _lib)
    from paper_2109_01158_b200.models import LameParams, fm_model_struct
    m = fm_model_struct(NeoHookean(ElasticParams(E=2e8, nu=0.3), dim=3))
    assert m.kind == _lib.FM_MODEL_NEOHOOKEAN and m.dim == 3
    m = fm_model_struct(NeoHookean(LameParams(1.0, 2.0), dim=2))
    assert (m.C1, m.D1) == (1.0, 2.0)
    m = fm_model_struct(PLaplacian(PLaplaceParams(p=1.8), dim=2))
    assert m.kind == _lib.FM_MODEL_PLAPLACE and m.p == 1.8

    class MyNH(NeoHookean):
        def density(self, F):
            return 0.0

    with pytest.raises(NotImplementedError):
        fm_model_struct(MyNH(ElasticParams(E=1.0, nu=0.3), dim=2))

    class Duck:
        d, dim = 1, 2
        params = PLaplaceParams(p=3.0)

        def density(self, G):
            return 0.0

    with pytest.raises(NotImplementedError):
        fm_model_struct(Duck())
    nh = NeoHookean(ElasticParams(E=1.0, nu=0.3), dim=2)
    nh.density = lambda F: 0.0
    with pytest.raises(NotImplementedError):
        fm_model_struct(nh)


def test_reference_model_objects_accepted():
    """The reference's own NeoHookean / PLaplacian (femmin.models) dispatch to
    the same kernels (drop-in: callers keep their model objects)."""
    ref = "/root/reference/pkg/src"
    if not os.path.isdir(ref):
        pytest.skip("reference not present (GPU box)")
    import sys
    sys.path.insert(0, ref)
    try:
        import femmin.models as fmm
    finally:
        sys.path.remove(ref)
    from paper_2109_01158_b200 import _lib
    from paper_2109_01158_b200.models import fm_model_struct
    m = fm_model_struct(fmm.NeoHookean(fmm.ElasticParams(E=2e8, nu=0.3), dim=3))
    p = fmm.ElasticParams(E=2e8, nu=0.3)
    assert m.kind == _lib.FM_MODEL_NEOHOOKEAN and (m.C1, m.D1) == (p.C1, p.D1)
    m = fm_model_struct(fmm.PLaplacian(fmm.PLaplaceParams(p=3.0), dim=2))
    assert m.kind == _lib.FM_MODEL_PLAPLACE and m.p == 3.0


def test_device_argument_checks_on_cpu_tensors():
    """Raw pointers reach the kernels only after a checked() pass: host
    tensors, wrong dtypes or lengths raise ValueError (never an assert)."""
    import torch
    from paper_2109_01158_b200._device import checked, ptr
    with pytest.raises(ValueError, match="CUDA"):
        checked(torch.zeros(3, dtype=torch.float64), "v", 3)
    with pytest.raises(ValueError, match="torch"):
        checked([0.0] * 3, "v", 3)
    with pytest.raises(ValueError):
        ptr(torch.zeros(3))
    assert checked(None, "b", 5) is None
