"""One small run of every evaluation kernel for compute-sanitizer (one tool per
call): fused J + gradient with several tiles per CTA, gradient only, energy,
FD, exact HVP, descent step, finishing pass."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2109_01158_b200 import problems  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 96
for pr in (problems.beam(n, n // 2, n // 2, seed=3), problems.lshape(6, 3.0, seed=3)):
    dm, model, b, v = pr.dm, pr.model, pr.b, pr.v
    J = torch.empty(3, dtype=torch.float64, device="cuda")
    g = dm.exact_gradient(v, model, b, J=J)
    dm.exact_gradient(v, model, b, g=g)
    dm.energy(v, model, b)
    dm.numeric_gradient(v, model, b, 1e-8 if dm.d == 3 else 1e-6)
    p = torch.zeros_like(v)
    dm.hvp(v, p, model)
    vd = v.clone()
    dm.descent(vd, model, b, 1e-12, 2)
    dm.check()
    torch.cuda.synchronize()
    print(pr.name, "tiles", dm.stats["n_tiles"], "J", float(J[0]))
