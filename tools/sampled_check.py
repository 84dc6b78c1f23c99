"""Sampled-dof parity at full size: the fused J + gradient of a
config (or one rank's x1-slab of config 5) against the oracle's per-dof
restatement of gradients.py:124-149 at N random free dofs.

    python tools/sampled_check.py cfg5 1/8 [N]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import femmin_oracle as O  # noqa: E402
from paper_2109_01158_b200 import problems  # noqa: E402
from paper_2109_01158_b200.parallel import slab_range  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
shard = sys.argv[2] if len(sys.argv) > 2 else ""
n = int(sys.argv[3]) if len(sys.argv) > 3 else 20000
t0 = time.time()
if cfg == "cfg5":
    r, w = (int(x) for x in shard.split("/"))
    ix0, ix1 = slab_range(1024, r, w)
    pr = problems.beam(1024, 512, 512, seed=2109, ix0=ix0, ix1=ix1, keep=True)
else:
    pr = problems.CONFIGS[cfg](keep=True)
dm, model, b, v = pr.dm, pr.model, pr.b, pr.v
J = torch.empty(3, dtype=torch.float64, device="cuda")
g = dm.exact_gradient(v, model, b, J=J)
Je = dm.energy(v, model, b).clone()
dm.check()
mt = pr.meta
rng = np.random.default_rng(21)
sample = np.sort(rng.choice(mt["dofs_minim"].numel(), size=n, replace=False))
dm_ = mt["dofs_minim"][torch.as_tensor(sample, device="cuda")]
nodes = torch.unique(dm_ // dm.d)
# only the sampled nodes' patches leave the device
prefix = mt["p_prefix"]
nm = mt["nodes_minim"]
rank = torch.searchsorted(nm, nodes)
lo = torch.where(rank > 0, prefix[(rank - 1).clamp(min=0)], torch.zeros_like(rank))
hi = prefix[rank]
rows = torch.cat([torch.arange(a, z, device="cuda") for a, z in zip(lo.tolist(), hi.tolist())])
el = mt["p_elems"][rows]
uel, inv = torch.unique(el, return_inverse=True)
conn = mt["conn"][uel].cpu().numpy()
vol = mt["volumes"][uel].cpu().numpy()
dphi = [x for x in mt["dphi"][:, uel].cpu().numpy()]
# local patch CSR over the sampled nodes only
lens = (hi - lo).cpu().numpy()
lprefix = np.cumsum(lens)
lelems = inv.cpu().numpy()
lslot = mt["p_slot"][rows].cpu().numpy()
dim = mt["coords"].shape[1]
omodel = (O.Model("nh", O.LameParams(model.params.C1, model.params.D1), dim) if dm.d > 1
          else O.Model("plap", O.PParams(model.params.p), dim))
q = dm_.cpu().numpy()
nodes_h = nodes.cpu().numpy()
local_dofs = np.searchsorted(nodes_h, q // dm.d) * dm.d + q % dm.d
vh = v.cpu().numpy()
bh = b.cpu().numpy()
# renumber: the oracle takes node-indexed v / b, so pass the global arrays with
# global connectivity and the sampled nodes as the "free" list
gs = O.sampled_exact_gradient(vh, conn, vol, dphi, lprefix, lelems, lslot, nodes_h, dm.d, omodel,
                              bh, q, np.arange(q.size))
gg = g.cpu().numpy()
err = np.abs(gg[sample] - gs).max() / np.abs(gg).max()
print(f"{cfg} {shard}: ne={pr.ne:,} J={float(J[0]):.12e} |J-J_energy|/|J|="
      f"{abs(float(J[0] - Je[0])) / abs(float(Je[0])):.1e}  sampled dofs {n}: "
      f"max|g - g_oracle| / max|g| = {err:.2e}  ({time.time() - t0:.0f} s)")
assert err < 1e-10

# nodal-patch FD at the sampled nodes: the direct-sum oracle on the sub-mesh of
# their patches (global node ids, only the sampled nodes free), bound
# 64 u sum_patch vol (|W+-| + L+-) / (2 eps) as in tests/test_gpu_parity.py
eps = 1e-8 if dm.d > 1 else 1e-6
gfd = dm.numeric_gradient(v, model, b, eps).cpu().numpy()
dm.check()
d = dm.d
sub_dofs = (nodes_h[:, None] * d + np.arange(d)[None]).ravel()
sub = O.OMesh(dim, -1, None, conn, vol, dphi, d, np.zeros(0, np.int64), nodes_h,
              np.zeros(0, np.int64), sub_dofs, np.arange(sub_dofs.size))
P = O.OPatches(lens, lelems, lslot, lprefix)
gd, scale = O.numeric_gradient_direct(vh, sub, P, omodel, bh, eps)
pos = np.searchsorted(mt["dofs_minim"].cpu().numpy(), sub_dofs)
ratio = np.abs(gfd[pos] - gd) / (64.0 * scale + 1e-300)
print(f"    FD at the {nodes_h.size} sampled nodes ({sub_dofs.size} dofs): max |g - g_direct| / bound "
      f"= {ratio.max():.2e}  ({time.time() - t0:.0f} s)")
assert ratio.max() <= 1.0
