"""Phase accounting of the warp-specialised fused kernel (profiling aid).

    python tools/ws_trace.py [--config cfg4] [--build-only]

Builds lib/libfemmin_wstrace.so with -DFM_WS_KERNEL=1 -DFM_WS_TRACE=1 (fm_eval_ws.cu, the warp-specialised kernel experiment): every
warp of CTAs 0..3 sums the clock64 cycles of each phase of its role over one
launch.  Prints, per role, the mean cycles per chunk of each phase.
Element groups: 0 loop overhead, 1 node-value wait, 2 record wait, 3 record
loads, 4 group barrier (+ next request), 5 element math, 6 staging-buffer
wait, 7 staging stores.  Node group: 0 loop overhead, 1 tile-start barrier +
gather issue, 2 node-value / table wait, 3 chunk head, 4 wait for the element
group, 5 own-entry sums, 6 cross items, 7 tile end.
"""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
LIB = os.path.join(ROOT, "paper_2109_01158_b200", "lib", "libfemmin_wstrace.so")
os.environ["FM_LIB_OVERRIDE"] = LIB
os.environ["FM_WS"] = "1"

from paper_2109_01158_b200 import build as B  # noqa: E402
CTAS, WARPS, PH = 4, 25, 8


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--build-only", action="store_true")
    args = ap.parse_args()
    if args.build_only or not os.path.exists(LIB):
        B.build_variant("wstrace", ["-DFM_WS_KERNEL=1", "-DFM_WS_TRACE=1"])
        if args.build_only:
            return
    import ctypes as C

    import numpy as np
    import torch

    from paper_2109_01158_b200 import _lib, problems
    pr = problems.CONFIGS[args.config]()
    g = torch.empty(pr.dm.nfree_dofs, dtype=torch.float64, device="cuda")
    J = torch.empty(3, dtype=torch.float64, device="cuda")
    for _ in range(3):
        pr.dm.exact_gradient(pr.v, pr.model, pr.b, g=g, J=J)
    torch.cuda.synchronize()
    lib = _lib.load()
    n = CTAS * WARPS * PH
    buf = (C.c_longlong * n)()
    lib.fm_ws_trace_copy.restype = C.c_int
    assert lib.fm_ws_trace_copy(buf, n) == 0
    a = np.frombuffer(buf, dtype=np.int64).reshape(CTAS, WARPS, PH).astype(np.float64)
    st = pr.dm.stats
    n_sm = torch.cuda.get_device_properties(0).multi_processor_count
    chunks = pr.dm.ne / 256 / n_sm  # approx. chunks per CTA
    print(f"{args.config}: ~{chunks:.0f} chunks per CTA, tiles {st['n_tiles']}")
    names = ["node group (warps 0-7)", "element group 0 (warps 8-15)",
             "element group 1 (warps 16-23)"]
    for r in range(3):
        m = a[:, 8 * r:8 * r + 8, :].mean(axis=(0, 1))
        tot = m.sum()
        print(f"{names[r]}: total {tot / 1e3:.0f} kcycles; per CTA-chunk: "
              + "  ".join(f"{k}:{m[k] / chunks:.0f}" for k in range(PH)))


if __name__ == "__main__":
    main()
