"""Race detector by repetition (compute-sanitizer is unavailable on the GPU
pool): every evaluation kernel run many times at a size with many tiles per
CTA must return bit-identical results."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2109_01158_b200 import problems  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
for name, pr in (("cfg4", problems.CONFIGS["cfg4"]()), ("cfg2", problems.CONFIGS["cfg2"]()),
                 ("cfg3", problems.CONFIGS["cfg3"]())):
    dm, model, b, v = pr.dm, pr.model, pr.b, pr.v
    J = torch.empty(3, dtype=torch.float64, device="cuda")
    p = torch.rand(v.shape, dtype=torch.float64, device="cuda") * (v != 0)
    ref = None
    bad = 0
    for r in range(reps):
        g = dm.exact_gradient(v, model, b, J=J).clone()
        J0 = J.clone()
        go = dm.exact_gradient(v, model, b).clone()
        E = dm.energy(v, model, b).clone()
        hp = dm.hvp(v, p, model).clone()
        fd = dm.numeric_gradient(v, model, b, 1e-8 if dm.d > 1 else 1e-6).clone() if r < 5 else None
        cur = (g, J0, go, E, hp, fd)
        if ref is None:
            ref = cur
        else:
            for a, c in zip(ref, cur):
                if a is not None and c is not None and not torch.equal(a, c):
                    bad += 1
    dm.check()
    print(name, "reps", reps, "mismatches", bad, flush=True)
    del pr
    torch.cuda.empty_cache()
