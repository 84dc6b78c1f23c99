"""Debug helper: run the fused kernel once on a small beam (used with
compute-sanitizer and the FM_TILE_ABLATE profiling knob)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2109_01158_b200 import problems

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 32
pr = problems.beam(nx, nx // 2, nx // 2, seed=1)
J = torch.empty(3, dtype=torch.float64, device="cuda")
for _ in range(3):
    g = pr.dm.exact_gradient(pr.v, pr.model, pr.b, J=J)
torch.cuda.synchronize()
print("ok", float(J[0]), float(g.abs().max()))
