"""Time (and, under ncu, profile) the exact Hessian-vector product at cfg4."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2109_01158_b200 import problems  # noqa: E402

pr = problems.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg4"]()
p = torch.rand(pr.v.shape, dtype=torch.float64, device="cuda") * (pr.v != 0)
out = torch.empty(pr.dm.nfree_dofs, dtype=torch.float64, device="cuda")
for _ in range(3):
    pr.dm.hvp(pr.v, p, pr.model, out=out)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    pr.dm.hvp(pr.v, p, pr.model, out=out)
b.record()
torch.cuda.synchronize()
pr.dm.check()
print(f"hvp {a.elapsed_time(b) / 20:.3f} ms")
