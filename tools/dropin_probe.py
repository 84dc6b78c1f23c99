"""Time the stages of the numpy drop-in call energy_and_gradient at cfg4
(profiling aid): upload (to_dev), fused kernel, download (to_host), whole call."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2109_01158_b200 as fb  # noqa: E402
from paper_2109_01158_b200 import problems  # noqa: E402
from paper_2109_01158_b200._device import to_dev, to_host  # noqa: E402
from paper_2109_01158_b200.patches import build_patches_device  # noqa: E402

pr = problems.beam(256, 128, 128, seed=2109)
hm = fb.generate_beam_mesh_3d(256, 128, 128)
hm = fb.mark_dirichlet(hm, fb.DirichletSpec([fb.DirichletRegion(where=lambda x: x[:, 0] < 1e-9)]),
                       d=3)
pfx, pel, psl = build_patches_device(torch.as_tensor(hm.elems2nodes).cuda(),
                                     torch.as_tensor(hm.nodes_minim).cuda(), hm.nn, 4)
hp = fb.Patches(lengths=np.diff(pfx.cpu().numpy(), prepend=0), elems=pel.cpu().numpy(),
                volumes=None, elems2nodes=None, dphi=None, logical=None,
                prefix=pfx.cpu().numpy(), slot=psl.cpu().numpy())
del pfx, pel, psl
load = fb.LinearLoad(b=pr.b.cpu().numpy())
v = pr.v.cpu().numpy().copy()
fb.energy_and_gradient(v, hm, hp, pr.model, load)


def t(fn, n=10):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


up = t(lambda: to_dev(v))
vd = to_dev(v)
g = torch.empty(pr.dm.nfree_dofs, dtype=torch.float64, device="cuda")
down = t(lambda: to_host(g))
call = t(lambda: fb.energy_and_gradient(v, hm, hp, pr.model, load))
print(f"upload {up:.2f} ms, download {down:.2f} ms, whole call {call:.2f} ms "
      f"(threads {os.cpu_count()})")

if "--profile" in sys.argv:
    import cProfile
    import pstats
    pr_ = cProfile.Profile()
    pr_.enable()
    for _ in range(5):
        fb.energy_and_gradient(v, hm, hp, pr.model, load)
    pr_.disable()
    pstats.Stats(pr_).sort_stats("tottime").print_stats(14)
