"""Time the FD gradient (and the fused exact pass) on the named configs."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2109_01158_b200 import problems

for name in sys.argv[1:]:
    pr = problems.CONFIGS[name]()
    eps = 1e-6 if name.startswith("cfg2") or name == "cfg1" else 1e-8
    g = torch.empty(pr.dm.nfree_dofs, dtype=torch.float64, device="cuda")
    def t(fn, n):
        fn(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(n): fn()
        b.record(); torch.cuda.synchronize()
        return a.elapsed_time(b) / n
    fd = t(lambda: pr.dm.numeric_gradient(pr.v, pr.model, pr.b, eps, g=g), 5)
    pr.dm.check()
    print(f"{name}: FD {fd:.3f} ms ({pr.ne / fd / 1e3:.0f} Melem/s)", flush=True)
    del pr
    torch.cuda.empty_cache()
