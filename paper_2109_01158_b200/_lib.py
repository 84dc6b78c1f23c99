"""ctypes binding of the C ABI in include/femmin_b200.h.

The shared library is built in-tree (``paper_2109_01158_b200/lib``) by
``build.py``.  There is no CPU fallback: importing the evaluation API without
the library, or calling it without a CUDA device, raises immediately.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# FM_LIB_OVERRIDE: profiling builds of the same library (tools/trace_exact.py)
LIB_PATH = os.environ.get("FM_LIB_OVERRIDE") or os.path.join(_HERE, "lib", "libfemmin_b200.so")

FM_OK, FM_INADMISSIBLE, FM_INVALID_ARG, FM_CUDA_ERROR, FM_DEGENERATE, FM_PATCH_STRUCTURE = range(6)
FM_MODEL_PLAPLACE, FM_MODEL_NEOHOOKEAN = 0, 1

i32, i64, u64, dbl, vp = C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_void_p
P64 = C.POINTER(C.c_int64)


class FmModel(C.Structure):
    _fields_ = [("kind", i32), ("dim", i32), ("p", dbl), ("C1", dbl), ("D1", dbl)]


class FmMeshDesc(C.Structure):
    _fields_ = [("dim", i32), ("d", i32), ("nn", i64), ("ne", i64), ("coords", vp),
                ("conn", vp), ("volumes", vp), ("dphi", vp), ("nfree", i64),
                ("nodes_minim", vp), ("fixed", vp), ("p_prefix", vp), ("p_elems", vp),
                ("p_slot", vp), ("p_total", i64)]


class FmTiling(C.Structure):
    _fields_ = [("tile_nodes", i32), ("box", i32 * 3)]


class FmCtxStats(C.Structure):
    _fields_ = [("n_tiles", i64), ("n_orphan_tiles", i64), ("tile_elems_total", i64),
                ("node_entries_total", i64), ("max_tile_elems", i64),
                ("max_tile_entries", i64), ("bytes_device", i64), ("redundancy", dbl),
                ("tile_threads", i32), ("ctas_per_sm", i32), ("node_bufs", i32),
                ("table_bufs", i32), ("entry_cap", i32), ("closure_cap", i32),
                ("cross_entries", i64), ("dict_tiles", i64)]


# name: (restype, argtypes) — every symbol declared in include/femmin_b200.h
SIGNATURES = {
    "fm_last_error": (C.c_char_p, []),
    "fm_version": (C.c_int, []),
    "fm_lshape_sizes": (C.c_int, [C.c_int, P64, P64]),
    "fm_gen_lshape": (C.c_int, [C.c_int, vp, vp, vp]),
    "fm_gen_rect": (C.c_int, [C.c_int, C.c_int, dbl, dbl, dbl, dbl, vp, vp, vp]),
    "fm_gen_beam": (C.c_int, [C.c_int, C.c_int, C.c_int, C.POINTER(dbl), C.c_int, C.c_int, vp, vp,
                             vp]),
    "fm_p1_gradients": (C.c_int, [C.c_int, i64, i64, vp, vp, vp, vp, P64, vp]),
    "fm_dirichlet_predicate": (C.c_int, [C.c_int, C.c_int, C.c_int, i64, vp, C.c_int, dbl, dbl,
                                         C.POINTER(i32), C.c_int, vp, P64, vp]),
    "fm_mark_dirichlet": (C.c_int, [i64, C.c_int, vp, vp, vp, vp, vp, vp, P64, vp]),
    "fm_build_patches": (C.c_int, [i64, i64, C.c_int, vp, vp, i64, vp, vp, vp, vp, P64, P64,
                                   vp]),
    "fm_load_constant": (C.c_int, [C.c_int, C.c_int, i64, i64, vp, vp, C.POINTER(dbl), vp, vp]),
    "fm_load_nodal": (C.c_int, [C.c_int, C.c_int, i64, i64, vp, vp, vp, vp, vp]),
    "fm_density_rows": (C.c_int, [C.POINTER(FmModel), i64, vp, vp, vp, P64, vp]),
    "fm_det_rows": (C.c_int, [C.c_int, i64, vp, vp, vp, vp]),
    "fm_eval_F": (C.c_int, [C.c_int, C.c_int, i64, vp, vp, vp, vp]),
    "fm_dot": (C.c_int, [i64, vp, vp, vp, vp]),
    "fm_segment_sums": (C.c_int, [i64, vp, vp, vp, vp]),
    "fm_field_uniform": (C.c_int, [i64, vp, i64, vp, u64, vp, vp]),
    "fm_field_nh": (C.c_int, [i64, C.c_int, vp, vp, i64, vp, u64, dbl, vp, vp]),
    "fm_ctx_create": (C.c_int, [C.POINTER(FmMeshDesc), C.POINTER(FmTiling), vp,
                                C.POINTER(vp)]),
    "fm_ctx_destroy": (C.c_int, [vp]),
    "fm_ctx_stats_get": (C.c_int, [vp, C.POINTER(FmCtxStats)]),
    "fm_energy": (C.c_int, [vp, C.POINTER(FmModel), vp, vp, vp, vp, vp]),
    "fm_grad_exact": (C.c_int, [vp, C.POINTER(FmModel), vp, vp, vp, vp, vp]),
    "fm_grad_fd": (C.c_int, [vp, C.POINTER(FmModel), vp, vp, dbl, vp, vp]),
    "fm_hvp_exact": (C.c_int, [vp, C.POINTER(FmModel), vp, vp, vp, vp]),
    "fm_descent_step": (C.c_int, [vp, vp, vp, dbl, vp]),
    "fm_descent": (C.c_int, [vp, C.POINTER(FmModel), vp, vp, dbl, C.c_int, vp, vp, vp]),
    "fm_comm_unique_id": (C.c_int, [vp]),
    "fm_slab_create": (C.c_int, [vp, C.c_int, C.c_int, i64, vp, vp, vp]),
    "fm_slab_reduce": (C.c_int, [vp, vp, vp, vp]),
    "fm_slab_destroy": (C.c_int, [vp]),
    "fm_stack_reduce": (C.c_int, [i64, vp, vp, vp, vp, C.c_int, vp, vp]),
    "fm_cg_scratch_doubles": (C.c_int, []),
    "fm_cg_init": (C.c_int, [i64, vp, vp, vp, vp, vp, vp, vp, vp]),
    "fm_cg_embed": (C.c_int, [vp, vp, vp, vp, C.c_int, dbl, vp, vp]),
    "fm_cg_iterate": (C.c_int, [i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "fm_ctx_check": (C.c_int, [vp, vp, P64]),
    "fm_hessian_pattern": (C.c_int, [i64, i64, C.c_int, C.c_int, vp, i64, vp, vp, vp, P64, vp]),
    "fm_color_d2": (C.c_int, [i64, vp, vp, vp, C.POINTER(i32), vp]),
    "fm_hess_perturb": (C.c_int, [i64, vp, vp, C.c_int, dbl, vp, vp]),
    "fm_hess_scatter": (C.c_int, [i64, vp, vp, vp, C.c_int, vp, vp, dbl, vp, vp]),
    "fm_hess_symmetrize": (C.c_int, [i64, vp, vp, vp, vp, vp]),
    "fm_ctx_launches": (i64, [vp]),
    "fm_ctx_time_next": (C.c_int, [vp, vp, vp]),
}

_lib = None


def load() -> C.CDLL:
    """Load the CUDA library (building it first if it is missing)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        from . import build as _build
        _build.build()
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class FemminCudaError(RuntimeError):
    pass


def last_error() -> str:
    return load().fm_last_error().decode()


def check(status: int, what: str = ""):
    """Map a C status to the reference's exception classes."""
    if status == FM_OK:
        return
    msg = last_error()
    if status == FM_INADMISSIBLE:
        from .models import InadmissibleStateError
        raise InadmissibleStateError(msg)
    if status == FM_DEGENERATE:
        from .mesh import DegenerateElementError
        raise DegenerateElementError(msg)
    if status == FM_PATCH_STRUCTURE:
        from .patches import PatchStructureError
        raise PatchStructureError(msg)
    if status == FM_INVALID_ARG:
        raise ValueError(msg)
    raise FemminCudaError(f"{what}: {msg}" if what else msg)
