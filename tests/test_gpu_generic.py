"""GPU parity on meshes that are NOT the structured benchmark grids, the
standalone helpers, admissibility at det F = 0, the tiling fallback and the
boundary's argument checks.

* the reference's unstructured hole mesh (mesh.py:246-286, bench.hole_problem)
  and a randomly renumbered Kuhn beam, both from golden files written by the
  reference itself (tests/golden/make_golden.py), and a larger renumbered
  beam against the oracle;
* gather / evaluate_F / segment_sums / linear_term / nodal LinearLoad /
  mass matrix (assembly.py:27-91, patches.py:74-83) against golden outputs;
* flattened elements (det F = 0 in exact arithmetic, a few ulps either way
  in numpy): J = +inf and the exact path's raise decided as the reference
  decides (models.py:59-71, 94-110).

Bars: J 1e-10 relative, exact gradient 1e-10 of max|g|, index structures
bit-exact, FD within the per-dof roundoff bound of the direct-sum oracle
(factor 64, as test_gpu_parity) and within 2x the reference FD's deviation.
"""

import numpy as np
import pytest

from oracle import femmin_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2109_01158_b200 as fb  # noqa: E402
from paper_2109_01158_b200 import device as fdev  # noqa: E402

J_TOL = 1e-10
G_TOL = 1e-10
FD_FACTOR = 64.0      # as tests/test_gpu_parity.py
FD_DEV_FACTOR = 1.5


def _mesh(g, pre=""):
    return fb.Mesh(dim=int(g[pre + "coords"].shape[1]), level=-1,
                   nodes2coord=g[pre + "coords"], elems2nodes=g[pre + "conn"],
                   volumes=g[pre + "volumes"], dphi=list(g[pre + "dphi"]), d=int(g[pre + "d"]),
                   nodes_dirichlet=g[pre + "nodes_dirichlet"], nodes_minim=g[pre + "nodes_minim"],
                   dofs_dirichlet=g[pre + "dofs_dirichlet"], dofs_minim=g[pre + "dofs_minim"],
                   dofs_minim_local=g[pre + "dofs_minim_local"])


def _omesh(g, pre=""):
    return O.OMesh(int(g[pre + "coords"].shape[1]), -1, g[pre + "coords"], g[pre + "conn"],
                   g[pre + "volumes"], list(g[pre + "dphi"]), int(g[pre + "d"]),
                   g[pre + "nodes_dirichlet"], g[pre + "nodes_minim"], g[pre + "dofs_dirichlet"],
                   g[pre + "dofs_minim"], g[pre + "dofs_minim_local"])


def _grel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def _evaluate_against(m, model, load, ref, om, omodel, eps):
    """Drop-in calls on the GPU vs the reference's own outputs (golden)."""
    pt = fb.build_patches(m)
    J, W = fb.energy(ref["v"], m, model, load)
    assert abs(J - ref["J"]) <= J_TOL * abs(ref["J"])
    np.testing.assert_allclose(W, ref["densities"], rtol=1e-12,
                               atol=1e-14 * np.abs(ref["densities"]).max())
    ge = fb.exact_gradient(ref["v"], m, pt, model, load)
    assert _grel(ge, ref["g_exact"]) < G_TOL
    Jf, gf = fb.energy_and_gradient(ref["v"], m, pt, model, load)
    assert abs(Jf - ref["J"]) <= J_TOL * abs(ref["J"]) and _grel(gf, ref["g_exact"]) < G_TOL
    gn = fb.numeric_gradient(ref["v"], m, pt, model, load, eps=eps)
    op = O.build_patches(om)
    gd, scale = O.numeric_gradient_direct(ref["v"], om, op, omodel, ref["b"], eps)
    ratio = np.abs(gn - gd) / (FD_FACTOR * scale + 1e-300)
    assert ratio.max() <= 1.0, ratio.max()
    gmax = np.abs(ref["g_exact"]).max()
    dev = np.abs(ref["g_fd"] - ref["g_exact"]).max() / gmax
    assert np.abs(gn - ref["g_fd"]).max() / gmax <= 2 * dev + 1e-12
    # no farther from the reference's exact gradient than the oracle's own FD
    assert (np.abs(gn - ref["g_exact"]).max()
            <= FD_DEV_FACTOR * np.abs(gd - ref["g_exact"]).max() + 1e-300)
    return pt


def test_hole_mesh_neohookean(golden):
    """The reference's unstructured domain: P1 data, partitions and patches
    on the GPU bit-exact / to rounding, evaluation against the reference."""
    g = golden("hole2")
    vol, dphi = fb.compute_p1_gradients(g["coords"], g["conn"])
    np.testing.assert_allclose(vol, g["volumes"], rtol=1e-12)
    assert np.abs(np.stack(dphi) - g["dphi"]).max() <= 1e-12 * np.abs(g["dphi"]).max()
    m = _mesh(g)
    spec = fb.DirichletSpec([fb.DirichletRegion(where=lambda x: x[:, 1] < 1e-9),
                             fb.DirichletRegion(where=lambda x: x[:, 0] < 1e-9)])
    raw = fb.Mesh(dim=2, level=-1, nodes2coord=g["coords"], elems2nodes=g["conn"],
                  volumes=g["volumes"], dphi=list(g["dphi"]), d=2)
    mm = fb.mark_dirichlet(raw, spec, d=2)
    for k in ("nodes_dirichlet", "nodes_minim", "dofs_dirichlet", "dofs_minim",
              "dofs_minim_local"):
        np.testing.assert_array_equal(getattr(mm, k), g[k], err_msg=k)
    model = fb.NeoHookean(fb.LameParams(float(g["C1"]), float(g["D1"])), dim=2)
    load = fb.LinearLoad(b=g["b"])
    om = _omesh(g)
    omodel = O.Model("nh", O.LameParams(float(g["C1"]), float(g["D1"])), 2)
    pt = _evaluate_against(m, model, load, g, om, omodel, 1e-8)
    np.testing.assert_array_equal(pt.prefix, g["p_prefix"])
    np.testing.assert_array_equal(pt.elems, g["p_elems"])
    np.testing.assert_array_equal(pt.slot, g["p_slot"])


@pytest.mark.parametrize("p", [3.0, 1.8])
def test_hole_mesh_plaplace(golden, p):
    g = golden("hole2")
    m = _mesh(g, "pl_")
    pre = f"pl{p:g}_"
    ref = {k[len(pre):]: val for k, val in g.items() if k.startswith(pre)}
    model = fb.PLaplacian(fb.PLaplaceParams(p), dim=2)
    _evaluate_against(m, model, fb.LinearLoad(b=ref["b"]), ref, _omesh(g, "pl_"),
                      O.Model("plap", O.PParams(p), 2), 1e-6)


def test_renumbered_beam_golden(golden):
    """Randomly permuted node / element numbering and rotated vertex order."""
    g = golden("beam6x3x3_renumbered")
    m = _mesh(g)
    model = fb.NeoHookean(fb.LameParams(float(g["C1"]), float(g["D1"])), dim=3)
    om = _omesh(g)
    omodel = O.Model("nh", O.LameParams(float(g["C1"]), float(g["D1"])), 3)
    pt = _evaluate_against(m, model, fb.LinearLoad(b=g["b"]), g, om, omodel, 1e-8)
    np.testing.assert_array_equal(pt.elems, g["p_elems"])
    np.testing.assert_array_equal(pt.slot, g["p_slot"])


def test_renumbered_beam_large_vs_oracle_and_structured():
    """24x12x12 beam (20,736 tets, many tiles): renumbered vs the oracle on the
    same numbering, and vs the structured numbering mapped back (the engine's
    result must not depend on the numbering beyond summation order)."""
    rng = np.random.default_rng(11)
    om0, omodel, b0, v0 = O.problem_beam(24, 12, 12, seed=5)
    nn, ne = om0.nodes2coord.shape[0], om0.elems2nodes.shape[0]
    pn = rng.permutation(nn)
    inv = np.empty(nn, np.int64)
    inv[pn] = np.arange(nn)
    conn = inv[om0.elems2nodes][rng.permutation(ne)]
    rot = np.array([(0, 1, 2, 3), (1, 2, 0, 3), (2, 0, 1, 3), (0, 2, 3, 1), (3, 1, 0, 2)])
    conn = np.take_along_axis(conn, rot[rng.integers(0, 5, ne)], axis=1)
    coords = om0.nodes2coord[pn]
    om = O._assemble_mesh(3, -1, coords, conn)
    om = O.mark_dirichlet(om, O.fixed_mask(om, [(O.left_face, None)], 3), 3)
    dofmap = (3 * pn[:, None] + np.arange(3)[None]).ravel()  # new dof -> old dof
    v = v0[dofmap]
    b = O.load_vector(om, (0.0, 0.0, -2.5e7), 3)
    op = O.build_patches(om)
    m = fb.Mesh(dim=3, level=-1, nodes2coord=om.nodes2coord, elems2nodes=om.elems2nodes,
                volumes=om.volumes, dphi=list(om.dphi), d=3,
                nodes_dirichlet=om.nodes_dirichlet, nodes_minim=om.nodes_minim,
                dofs_dirichlet=om.dofs_dirichlet, dofs_minim=om.dofs_minim,
                dofs_minim_local=om.dofs_minim_local)
    pt = fb.build_patches(m)
    np.testing.assert_array_equal(pt.elems, op.elems)
    np.testing.assert_array_equal(pt.slot, op.slot)
    model = fb.NeoHookean(fb.LameParams(omodel.params.C1, omodel.params.D1), dim=3)
    load = fb.LinearLoad(b=b)
    Jf, gf = fb.energy_and_gradient(v, m, pt, model, load)
    Jo = O.energy(v, om, omodel, b)[0]
    go = O.exact_gradient(v, om, op, omodel, b)
    assert abs(Jf - Jo) <= J_TOL * abs(Jo) and _grel(gf, go) < G_TOL
    gn = fb.numeric_gradient(v, m, pt, model, load, eps=1e-8)
    gd, scale = O.numeric_gradient_direct(v, om, op, omodel, b, 1e-8)
    assert (np.abs(gn - gd) <= FD_FACTOR * scale + 1e-300).all()
    # structured numbering, mapped to the permuted free-dof order
    m0 = fb.Mesh(dim=3, level=-1, nodes2coord=om0.nodes2coord, elems2nodes=om0.elems2nodes,
                 volumes=om0.volumes, dphi=list(om0.dphi), d=3,
                 nodes_dirichlet=om0.nodes_dirichlet, nodes_minim=om0.nodes_minim,
                 dofs_dirichlet=om0.dofs_dirichlet, dofs_minim=om0.dofs_minim,
                 dofs_minim_local=om0.dofs_minim_local)
    J0, g0 = fb.energy_and_gradient(v0, m0, fb.build_patches(m0), model, fb.LinearLoad(b=b0))
    pos0 = np.full(3 * nn, -1)
    pos0[om0.dofs_minim] = np.arange(om0.dofs_minim.size)
    g0_perm = g0[pos0[dofmap[om.dofs_minim]]]
    assert abs(Jf - J0) <= 1e-12 * abs(J0) and _grel(gf, g0_perm) < 1e-12


def test_standalone_helpers_vs_reference(golden):
    g = golden("exports")
    for tag, d in (("l", 1), ("b", 3)):
        conn, V = g[f"{tag}_conn"], g[f"{tag}_V"]
        vals = fb.gather(V, conn)
        np.testing.assert_array_equal(np.stack(vals), g[f"{tag}_gather"])
        F = fb.evaluate_F(list(g[f"{tag}_dphi"]), vals)
        np.testing.assert_array_equal(np.array(F), g[f"{tag}_F"])   # einsum order, bit-exact
        seg = fb.segment_sums(g[f"{tag}_rows"], g[f"{tag}_indx"])
        ref = g[f"{tag}_segsum"]
        # direct fixed-order sums vs the reference's cumsum differences
        assert np.abs(seg - ref).max() <= 1e-12 * np.abs(g[f"{tag}_rows"]).sum()
        m = fb.Mesh(dim=int(g[f"{tag}_coords"].shape[1]), level=-1,
                    nodes2coord=g[f"{tag}_coords"], elems2nodes=conn,
                    volumes=g[f"{tag}_volumes"], dphi=list(g[f"{tag}_dphi"]), d=d)
        load = fb.LinearLoad.assemble(m, g[f"{tag}_f_nodal"], d=d)       # fm_load_nodal
        bref = g[f"{tag}_b_nodal"]
        assert np.abs(load.b - bref).max() <= 1e-13 * np.abs(bref).max()
        M = fb.assemble_mass_matrix(m)
        M.sort_indices()
        np.testing.assert_array_equal(M.indptr, g[f"{tag}_M_indptr"])
        np.testing.assert_array_equal(M.indices, g[f"{tag}_M_indices"])
        np.testing.assert_allclose(M.data, g[f"{tag}_M_data"], rtol=1e-15)
        lt = fb.linear_term(fb.LinearLoad(b=bref), g[f"{tag}_v"])         # fm_dot
        assert abs(lt - g[f"{tag}_linear_term"]) <= 1e-13 * np.abs(bref * g[f"{tag}_v"]).sum()


def test_degenerate_det_decisions(golden):
    """Flattened elements: the fused J + gradient and the energy kernel decide
    admissibility as the reference (+inf J, InadmissibleStateError)."""
    g = golden("degenerate_beam4x2x2")
    m = _mesh(g)
    pt = fb.build_patches(m)
    model = fb.NeoHookean(fb.LameParams(float(g["C1"]), float(g["D1"])), dim=3)
    dm = fdev.context_for(m, pt, 3)
    n_inf = 0
    for v, J, r in zip(g["v"], g["J"], g["raises"]):
        Je, _ = fb.energy(v, m, model)
        assert np.isinf(Je) == np.isinf(J)
        if not np.isinf(J):
            assert abs(Je - J) <= J_TOL * abs(J)
        vd = torch.from_numpy(v).cuda()
        Jd = torch.empty(3, dtype=torch.float64, device="cuda")
        dm.exact_gradient(vd, model, None, J=Jd)
        Jf = float(Jd[0])
        assert np.isinf(Jf) == np.isinf(J), (Jf, J)
        if not np.isinf(J):
            assert abs(Jf - J) <= J_TOL * abs(J)
        if r:
            with pytest.raises(fb.InadmissibleStateError):
                dm.check()
        else:
            dm.check()
        n_inf += bool(np.isinf(J))
    assert 0 < n_inf < len(g["J"])  # both outcomes are exercised


def test_tiling_capacity_fallback():
    """A tiling whose tiles exceed the per-tile caps (here > 9 chunks) is
    shrunk by the context build instead of failing; results agree with the
    default tiling to rounding."""
    om, omodel, b, v = O.problem_beam(24, 12, 12, seed=3)
    m = fb.Mesh(dim=3, level=-1, nodes2coord=om.nodes2coord, elems2nodes=om.elems2nodes,
                volumes=om.volumes, dphi=list(om.dphi), d=3,
                nodes_dirichlet=om.nodes_dirichlet, nodes_minim=om.nodes_minim,
                dofs_dirichlet=om.dofs_dirichlet, dofs_minim=om.dofs_minim,
                dofs_minim_local=om.dofs_minim_local)
    pt = fb.build_patches(m)
    model = fb.NeoHookean(fb.LameParams(omodel.params.C1, omodel.params.D1), dim=3)
    big = fb.DeviceMesh.from_host(m, pt, tiling=(256, (24, 24, 24)))
    ref = fb.DeviceMesh.from_host(m, pt)
    assert big.stats["n_tiles"] > 1
    vd, bd = torch.from_numpy(v).cuda(), torch.from_numpy(b).cuda()
    J1, J2 = (torch.empty(3, dtype=torch.float64, device="cuda") for _ in range(2))
    g1 = big.exact_gradient(vd, model, bd, J=J1).cpu().numpy()
    g2 = ref.exact_gradient(vd, model, bd, J=J2).cpu().numpy()
    assert _grel(g1, g2) < 1e-13 and abs(float(J1[0] - J2[0])) <= 1e-13 * abs(float(J2[0]))


def test_device_argument_checks():
    """Wrong dtype / length / device arguments raise ValueError before any
    pointer reaches a kernel."""
    om, omodel, b, v = O.problem_beam(4, 2, 2, seed=3)
    m = fb.Mesh(dim=3, level=-1, nodes2coord=om.nodes2coord, elems2nodes=om.elems2nodes,
                volumes=om.volumes, dphi=list(om.dphi), d=3,
                nodes_dirichlet=om.nodes_dirichlet, nodes_minim=om.nodes_minim,
                dofs_dirichlet=om.dofs_dirichlet, dofs_minim=om.dofs_minim,
                dofs_minim_local=om.dofs_minim_local)
    dm = fb.DeviceMesh.from_host(m, fb.build_patches(m))
    model = fb.NeoHookean(fb.LameParams(omodel.params.C1, omodel.params.D1), dim=3)
    vd = torch.from_numpy(v).cuda()
    with pytest.raises(ValueError, match="float64"):
        dm.exact_gradient(vd.float(), model)
    with pytest.raises(ValueError, match="elements"):
        dm.exact_gradient(vd[:-3].contiguous(), model)
    with pytest.raises(ValueError, match="elements"):
        dm.exact_gradient(vd, model, g=torch.empty(5, dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError, match="CUDA"):
        dm.energy(torch.from_numpy(v), model)
    with pytest.raises(ValueError):
        dm.hvp(vd, vd[:10].contiguous(), model)
    g = dm.exact_gradient(vd, model)
    assert g.numel() == om.dofs_minim.size


def test_drop_in_shares_one_context_per_mesh():
    """energy (no patches) and the gradients (the user's canonical Patches)
    use ONE device context; a non-canonical patch structure gets
    its own."""
    om, omodel, b, v = O.problem_beam(6, 3, 3, seed=4)
    m = fb.Mesh(dim=3, level=-1, nodes2coord=om.nodes2coord, elems2nodes=om.elems2nodes,
                volumes=om.volumes, dphi=list(om.dphi), d=3,
                nodes_dirichlet=om.nodes_dirichlet, nodes_minim=om.nodes_minim,
                dofs_dirichlet=om.dofs_dirichlet, dofs_minim=om.dofs_minim,
                dofs_minim_local=om.dofs_minim_local)
    pt = fb.build_patches(m)
    model = fb.NeoHookean(fb.LameParams(omodel.params.C1, omodel.params.D1), dim=3)
    before = len(fdev._CTX)
    fb.energy(v, m, model)
    fb.exact_gradient(v, m, pt, model)
    fb.numeric_gradient(v, m, pt, model)
    assert len(fdev._CTX) == before + 1
    # a hand-made (non-canonical) patch structure: reversed element order in patch 0
    el = pt.elems.copy()
    n0 = int(pt.prefix[0])
    el[:n0] = el[:n0][::-1]
    sl = pt.slot.copy()
    sl[:n0] = sl[:n0][::-1]
    pt2 = fb.Patches(lengths=pt.lengths, elems=el, volumes=None, elems2nodes=None, dphi=None,
                     logical=None, prefix=pt.prefix, slot=sl)
    g2 = fb.exact_gradient(v, m, pt2, model)
    assert len(fdev._CTX) == before + 2
    assert _grel(g2, fb.exact_gradient(v, m, pt, model)) < 1e-13
