import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from oracle import femmin_oracle as O
import paper_2109_01158_b200 as fb
from test_gpu_generic import _mesh, _omesh
def load(n):
    z = np.load(f'/root/repo/tests/golden/{n}.npz'); return {k: z[k] for k in z.files}
for name, eps in (("cfg1_lshape4_p3", 1e-6), ("lshape4_p1.8", 1e-6), ("rect32x16_nh", 1e-8), ("beam8x4x4_nh", 1e-8), ("hole2", 1e-8), ("beam6x3x3_renumbered", 1e-8)):
    g = load(name); m = _mesh(g); om = _omesh(g)
    if "C1" in g:
        dim = m.dim
        model = fb.NeoHookean(fb.LameParams(float(g["C1"]), float(g["D1"])), dim=dim)
        omodel = O.Model("nh", O.LameParams(float(g["C1"]), float(g["D1"])), dim)
    else:
        model = fb.PLaplacian(fb.PLaplaceParams(float(g["p"])), 2); omodel = O.Model("plap", O.PParams(float(g["p"])), 2)
    pt = fb.build_patches(m); load_ = fb.LinearLoad(b=g["b"])
    gn = fb.numeric_gradient(g["v"], m, pt, model, load_, eps=eps)
    op = O.build_patches(om)
    gd, scale = O.numeric_gradient_direct(g["v"], om, op, omodel, g["b"], eps)
    ge = g["g_exact"]; gm = np.abs(ge).max()
    print(f"{name}: max ratio to 64*scale {np.max(np.abs(gn-gd)/(64*scale+1e-300)):.3g}; "
          f"dev from exact: gpu {np.abs(gn-ge).max()/gm:.3g} oracle-direct {np.abs(gd-ge).max()/gm:.3g} reference {np.abs(g['g_fd']-ge).max()/gm:.3g}; "
          f"|gpu-ref| {np.abs(gn-g['g_fd']).max()/gm:.3g}")
