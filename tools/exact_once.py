"""A few fused J + exact gradient launches on a config (ncu target)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2109_01158_b200 import problems  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
pr = problems.CONFIGS[name]()
g = torch.empty(pr.dm.nfree_dofs, dtype=torch.float64, device="cuda")
J = torch.empty(3, dtype=torch.float64, device="cuda")
for _ in range(n):
    pr.dm.exact_gradient(pr.v, pr.model, pr.b, g=g, J=J)
pr.dm.check()
torch.cuda.synchronize()
print("ok", float(J[0]))
