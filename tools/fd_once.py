"""One FD gradient launch on a config (profiling target for ncu)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2109_01158_b200 import problems  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2
pr = problems.CONFIGS[name]()
eps = 1e-6 if name.startswith("cfg2") or name == "cfg1" else 1e-8
g = torch.empty(pr.dm.nfree_dofs, dtype=torch.float64, device="cuda")
for _ in range(n):
    pr.dm.numeric_gradient(pr.v, pr.model, pr.b, eps, g=g)
pr.dm.check()
torch.cuda.synchronize()
print("ok", float(g.abs().max()))
