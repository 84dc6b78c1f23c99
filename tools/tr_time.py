"""Wall time per gradient call of the device trust region at a config
(host-loop CG vs device-resident CG), against the gradient kernel alone.

    python tools/tr_time.py [cfg4] [iters]
"""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2109_01158_b200 import problems  # noqa: E402
from paper_2109_01158_b200.solver import SolveOptions, minimize_device  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
pr = problems.CONFIGS[name](keep=True)
dm, model, b, v = pr.dm, pr.model, pr.b, pr.v
g = torch.empty(dm.nfree_dofs, dtype=torch.float64, device="cuda")
for _ in range(3):
    dm.exact_gradient(v, model, b, g=g)
torch.cuda.synchronize()
a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    dm.exact_gradient(v, model, b, g=g)
z.record()
torch.cuda.synchronize()
kern = a.elapsed_time(z) / 20
print(f"{name}: gradient (no J) {kern:.3f} ms per call")
for hvp in ("fd", "exact"):
    for dev in (False, True):
        o = SolveOptions(max_iters=iters, max_cg=20, hvp=hvp, device_cg=dev)
        minimize_device(dm, model, b, v, pr.meta["dofs_minim"], SolveOptions(max_iters=1, max_cg=2, hvp=hvp, device_cg=dev))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = minimize_device(dm, model, b, v, pr.meta["dofs_minim"], o)
        t = time.perf_counter() - t0
        calls = r.n_grad + 2 * getattr(r, "n_hvp", 0)
        print(f"  hvp={hvp:5s} device_cg={dev!s:5s}: {t:.3f} s, {r.n_grad} grad + "
              f"{getattr(r, 'n_hvp', 0)} hvp calls, {t / max(1, calls) * 1e3:.3f} ms per "
              f"gradient-equivalent ({t / max(1, calls) * 1e3 / kern:.2f}x kernel), J {r.J_u:.10e}",
              flush=True)
