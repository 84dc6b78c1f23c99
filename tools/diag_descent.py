"""Diagnostic: J(v) from the energy kernel, the fused kernel and the first
descent iteration must agree (same v)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2109_01158_b200 import problems
nx = int(sys.argv[1]) if len(sys.argv) > 1 else 64
pr = problems.beam(nx, nx // 2, nx // 2, seed=2109)
dm, model, b, v = pr.dm, pr.model, pr.b, pr.v
Je = dm.energy(v, model, b).clone()
J = torch.empty(3, dtype=torch.float64, device="cuda")
g = dm.exact_gradient(v, model, b, J=J)
print("energy kernel", Je.tolist())
print("fused kernel ", J.tolist())
Jh = torch.empty((3, 3), dtype=torch.float64, device="cuda")
vd = v.clone()
dm.descent(vd, model, b, 1e-12, 3, J_hist=Jh)
print("descent J_hist", Jh.tolist())
dm.check()
v0 = v.clone()
for i in range(3):
    dm.exact_gradient(v, model, b, g=g, J=J)
    print("repeat fused", J.tolist(), torch.equal(v, v0))
