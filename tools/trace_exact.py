"""Phase timeline of the fused J + grad J tile kernel (profiling aid).

    python tools/trace_exact.py [--config cfg4] [--build-only]

Builds a separate library (lib/libfemmin_trace.so) with fm_eval_exact.cu
compiled under -DFM_TRACE=1: the warp leaders of CTAs 0..3 record clock64()
at the phase boundaries of every chunk:
  0 loop top   1 records arrived   2 compute + staging done   3 after barrier 1
  4 consume done   5 after barrier 2        (6 / 7: tile start / tables ready)
and prints the median / mean cycles of each phase per chunk.  The product
library is untouched; the traced one is selected through FM_LIB_OVERRIDE.
"""

from __future__ import annotations

import argparse
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
TRACE_LIB = os.path.join(ROOT, "paper_2109_01158_b200", "lib", "libfemmin_trace.so")
os.environ["FM_LIB_OVERRIDE"] = TRACE_LIB  # before the package reads its library path

from paper_2109_01158_b200 import build as B  # noqa: E402
CTAS, WARPS, CHUNKS, STAMPS = 4, 8, 160, 8


def build_trace():
    # every unit gets the define; only fm_eval_exact.cu uses it
    return B.build_variant("trace", ["-DFM_TRACE=1"])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--build-only", action="store_true")
    args = ap.parse_args()
    if args.build_only or not os.path.exists(TRACE_LIB):
        build_trace()
        if args.build_only:
            return
    import ctypes as C

    import numpy as np
    import torch

    from paper_2109_01158_b200 import _lib, problems
    pr = (problems.beam(256, 128, 128, seed=2109) if args.config == "cfg4"
          else problems.CONFIGS[args.config]())
    g = torch.empty(pr.dm.nfree_dofs, dtype=torch.float64, device="cuda")
    J = torch.empty(3, dtype=torch.float64, device="cuda")
    for _ in range(3):
        pr.dm.exact_gradient(pr.v, pr.model, pr.b, g=g, J=J)
    torch.cuda.synchronize()
    lib = _lib.load()
    n = CTAS * WARPS * CHUNKS * STAMPS
    buf = (C.c_longlong * n)()
    lib.fm_trace_copy.restype = C.c_int
    assert lib.fm_trace_copy(buf, n) == 0
    t = np.frombuffer(buf, dtype=np.int64).reshape(CTAS, WARPS, CHUNKS, STAMPS).astype(np.float64)
    names = ["wait records", "compute+stage", "barrier 1", "consume", "barrier 2"]
    for cta in range(CTAS):
        tt = t[cta]
        valid = (tt[:, :, 0] > 0) & (tt[:, :, 5] > 0)
        nchunk = int(valid[0].sum())
        print(f"CTA {cta}: {nchunk} chunks traced")
        rows = []
        for k in range(5):
            d = (tt[:, :, k + 1] - tt[:, :, k])[valid]
            rows.append((names[k], np.median(d), d.mean(), d.max()))
        nxt = (tt[:, 1:, 0] - tt[:, :-1, 5])[valid[:, 1:] & valid[:, :-1]]
        rows.append(("to next chunk", np.median(nxt), nxt.mean(), nxt.max()))
        per = np.diff(tt[0, :, 0][valid[0]])
        for name, med, mean, mx in rows:
            print(f"  {name:16s} median {med:8.0f}  mean {mean:8.0f}  max {mx:8.0f} cycles")
        print(f"  chunk period (warp 0): median {np.median(per):.0f} mean {per.mean():.0f}")
        st = tt[:, :, 7] - tt[:, :, 6]
        st = st[(tt[:, :, 6] > 0) & (tt[:, :, 7] > 0)]
        if st.size:
            print(f"  tile start (tables wait): median {np.median(st):.0f} mean {st.mean():.0f}")
        # per-warp compute spread (imbalance within the CTA)
        comp = (tt[:, :, 2] - tt[:, :, 1])
        cons = (tt[:, :, 4] - tt[:, :, 3])
        print("  per-warp mean compute:", " ".join(f"{x:.0f}" for x in comp[:, valid[0]].mean(1)))
        print("  per-warp mean consume:", " ".join(f"{x:.0f}" for x in cons[:, valid[0]].mean(1)))


if __name__ == "__main__":
    main()
