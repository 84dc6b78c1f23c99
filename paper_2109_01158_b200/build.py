"""Build the in-tree CUDA library ``lib/libfemmin_b200.so`` for sm_100a.

    python -m paper_2109_01158_b200.build        (or __graft_entry__.build())

Plain nvcc, one object per translation unit, relinked only when a source or
header changed.  Element arithmetic that must follow the reference's rounding
order uses explicit round-to-nearest intrinsics (fm_density.cuh), so every
unit compiles with FMA contraction on.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libfemmin_b200.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
BASE = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
        "--expt-relaxed-constexpr", f"-I{INCLUDE}", f"-I{CSRC}"]
UNITS = {
    "fm_prep.cu": [],
    "fm_ctx.cu": [],
    "fm_eval_exact.cu": [],
    "fm_eval_ws.cu": [],
    "fm_eval_ref.cu": [],
    "fm_hessian.cu": [],
    "fm_cg.cu": [],
    "fm_slab.cu": [],
}


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    return hs + [os.path.join(INCLUDE, "femmin_b200.h")]


def _compile(unit, extra, objdir, force):
    src = os.path.join(CSRC, unit)
    obj = os.path.join(objdir, unit.replace(".cu", ".o"))
    hdr_mtime = max(os.path.getmtime(h) for h in _headers())
    if (not force and os.path.exists(obj)
            and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_mtime)):
        return obj, None
    cmd = [_nvcc(), *ARCH, *BASE, *extra, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed on {unit}:\n{r.stdout}\n{r.stderr}")
    return obj, r.stdout + r.stderr


def _build(lib: str, objdir: str, defines: list[str], force: bool, verbose: bool) -> str:
    """Compile every unit (in parallel, only what changed) and link ``lib``."""
    os.makedirs(objdir, exist_ok=True)
    with ThreadPoolExecutor(max_workers=len(UNITS)) as ex:
        res = list(ex.map(lambda kv: _compile(kv[0], kv[1] + defines, objdir, force),
                          UNITS.items()))
    objs = [o for o, _ in res]
    log = [l for _, l in res if l is not None]
    if (force or log or not os.path.exists(lib)
            or os.path.getmtime(lib) < max(os.path.getmtime(o) for o in objs)):
        cmd = [_nvcc(), *ARCH, "-shared", "-o", lib, *objs, "-lcudart", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    if log:
        with open(os.path.join(objdir, "ptxas.log"), "w") as fh:
            fh.write("\n".join(log))
        if verbose:
            print("\n".join(log))
    return lib


def build(verbose: bool = False, force: bool = False) -> str:
    """The product library lib/libfemmin_b200.so."""
    os.makedirs(LIBDIR, exist_ok=True)
    return _build(LIB, os.path.join(LIBDIR, "obj"), [], force, verbose)


def build_variant(name: str, defines: list[str], force: bool = False) -> str:
    """A profiling build of the same sources (lib/libfemmin_<name>.so, e.g.
    -DFM_TRACE=1 or -DFM_ABLATE=1), selected at run time with FM_LIB_OVERRIDE;
    the product library never carries these switches."""
    os.makedirs(LIBDIR, exist_ok=True)
    return _build(os.path.join(LIBDIR, f"libfemmin_{name}.so"),
                  os.path.join(LIBDIR, f"obj_{name}"), defines, force, False)


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
