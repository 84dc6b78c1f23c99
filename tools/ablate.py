"""Time the fused tile kernel under FM_TILE_ABLATE settings (profiling aid;
ablated runs compute wrong results on purpose, so no checks are made).

    python tools/ablate.py 0 1 2 4 ...

The switches exist only in a separate profiling build (lib/libfemmin_ablate.so,
-DFM_ABLATE=1), selected through FM_LIB_OVERRIDE; the product library has none.
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, torch
sys.path.insert(0, %r)
from paper_2109_01158_b200 import problems
pr = problems.beam(256, 128, 128, seed=2109)
g = torch.empty(pr.dm.nfree_dofs, dtype=torch.float64, device="cuda")
J = torch.empty(3, dtype=torch.float64, device="cuda")
for _ in range(3):
    pr.dm.exact_gradient(pr.v, pr.model, pr.b, g=g, J=J)
torch.cuda.synchronize()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
for a, z in ev:  # materialise the CUDA events
    a.record(); z.record()
for a, z in ev:
    pr.dm.time_next(a, z)
    pr.dm.exact_gradient(pr.v, pr.model, pr.b, g=g, J=J)
torch.cuda.synchronize()
print(sum(a.elapsed_time(z) for a, z in ev) / len(ev))
''' % ROOT

sys.path.insert(0, ROOT)
from paper_2109_01158_b200 import build as B  # noqa: E402

LIB = B.build_variant("ablate", ["-DFM_ABLATE=1"])
for setting in sys.argv[1:]:
    env = dict(os.environ, FM_TILE_ABLATE=setting, FM_LIB_OVERRIDE=LIB)
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    out = r.stdout.strip().splitlines()
    print(f"ablate {setting}: kernel {out[-1] if out else 'FAILED ' + r.stderr[-300:]} ms")
