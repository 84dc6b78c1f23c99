"""Pin the CPU oracle against golden vectors produced by the real reference.

These run without a GPU.  Bit-exact (``assert_array_equal``) wherever the
oracle performs the same numpy operations as the reference; the few places
where only the summation order differs use tolerances written inline.
"""

import numpy as np
import pytest

from oracle import femmin_oracle as O


def _mesh_from_golden(g):
    m = O.OMesh(int(g["coords"].shape[1]), -1, g["coords"], g["conn"], g["volumes"],
                list(g["dphi"]), int(g["d"]), g["nodes_dirichlet"], g["nodes_minim"],
                g["dofs_dirichlet"], g["dofs_minim"], g["dofs_minim_local"])
    return m


def _patches_from_golden(g):
    return O.OPatches(g["p_lengths"], g["p_elems"], g["p_slot"], g["p_prefix"])


def _check_mesh(m, g, exact_geometry=True):
    np.testing.assert_array_equal(m.nodes2coord, g["coords"])
    np.testing.assert_array_equal(m.elems2nodes, g["conn"])
    if exact_geometry:
        np.testing.assert_array_equal(m.volumes, g["volumes"])
        np.testing.assert_array_equal(np.stack(m.dphi), g["dphi"])
    for k in ("nodes_dirichlet", "nodes_minim", "dofs_dirichlet", "dofs_minim",
              "dofs_minim_local"):
        if k in g:
            np.testing.assert_array_equal(getattr(m, k), g[k], err_msg=k)


def _check_patches(p, g):
    np.testing.assert_array_equal(p.lengths, g["p_lengths"])
    np.testing.assert_array_equal(p.prefix, g["p_prefix"])
    np.testing.assert_array_equal(p.elems, g["p_elems"])
    np.testing.assert_array_equal(p.slot, g["p_slot"])
    np.testing.assert_array_equal(O.prefix_indices(p, 3), g["p_indx3"])


@pytest.mark.parametrize("level", [0, 1, 2, 3])
def test_lshape_generator_bit_exact(golden, level):
    g = golden("lshape_meshes")
    m = O.lshape_mesh(level)
    np.testing.assert_array_equal(m.nodes2coord, g[f"lshape{level}_coords"])
    np.testing.assert_array_equal(m.elems2nodes, g[f"lshape{level}_conn"])
    np.testing.assert_array_equal(m.volumes, g[f"lshape{level}_volumes"])
    np.testing.assert_array_equal(np.stack(m.dphi), g[f"lshape{level}_dphi"])


def test_lshape_counts_match_reference_tests():
    # test_mesh.py:51-55 (level 0: 24 elements, 21 nodes)
    m = O.lshape_mesh(0)
    assert (m.ne, m.nn) == (24, 21)


def test_cfg1_problem_bit_exact(golden):
    g = golden("cfg1_lshape4_p3")
    m, model, b, v = O.problem_lshape(4, 3.0, seed=2109)
    _check_mesh(m, g)
    assert (m.ne, m.nn, m.dofs_minim.size) == (6144, 3201, 2945)
    p = O.build_patches(m)
    _check_patches(p, g)
    assert p.total_rows == 17670
    np.testing.assert_array_equal(v, g["v"])
    np.testing.assert_array_equal(b, g["b"])
    J, W = O.energy(v, m, model, b)
    assert J == g["J"]
    np.testing.assert_array_equal(W, g["densities"])
    np.testing.assert_array_equal(O.exact_gradient(v, m, p, model, b), g["g_exact"])
    np.testing.assert_array_equal(O.numeric_gradient(v, m, p, model, b, eps=1e-6), g["g_fd"])


def test_lshape_p18_bit_exact(golden):
    g = golden("lshape4_p1.8")
    m, model, b, v = O.problem_lshape(4, 1.8, seed=2110)
    p = O.build_patches(m)
    np.testing.assert_array_equal(v, g["v"])
    assert O.energy(v, m, model, b)[0] == g["J"]
    np.testing.assert_array_equal(O.exact_gradient(v, m, p, model, b), g["g_exact"])
    np.testing.assert_array_equal(O.numeric_gradient(v, m, p, model, b, 1e-6), g["g_fd"])


@pytest.mark.parametrize("p", [1.5, 3.0, 4.0])
def test_lshape1_reference_fixture(golden, p):
    g = golden("lshape1_plap")
    m = _mesh_from_golden(g)
    pt = _patches_from_golden(g)
    _check_patches(O.build_patches(m), g)
    model = O.Model("plap", O.PParams(p), 2)
    b = g[f"b_p{p:g}"]
    v = g["v"]
    assert O.energy(v, m, model, b)[0] == g[f"J_p{p:g}"]
    np.testing.assert_array_equal(O.exact_gradient(v, m, pt, model, b), g[f"g_exact_p{p:g}"])
    np.testing.assert_array_equal(O.numeric_gradient(v, m, pt, model, b, 1e-6), g[f"g_fd_p{p:g}"])
    # the loop oracle (test_gradients.py:133-155) agrees to 1e-13
    ge = O.exact_gradient(v, m, pt, model, None)
    np.testing.assert_allclose(ge, O.exact_gradient_loop(v, m, model), rtol=1e-12, atol=1e-12)


def test_bar_level1_bit_exact(golden):
    g = golden("bar1_nh")
    m = O.bar_mesh(0.4, 0.01, 0.01, 1)
    fixed = O.fixed_mask(m, [(lambda x: x[:, 0] < 1e-9, None),
                             (lambda x: x[:, 0] > 0.4 - 1e-9, None)], 3)
    m = O.mark_dirichlet(m, fixed, 3)
    _check_mesh(m, g)
    assert (m.nn, m.ne, m.nodes_dirichlet.size, m.dofs_minim.size) == (729, 1920, 18, 2133)
    p = O.build_patches(m)
    _check_patches(p, g)
    assert (p.lengths.size, p.total_rows) == (711, 7584)        # test_patches.py:14-16
    model = O.Model("nh", O.LameParams(float(g["C1"]), float(g["D1"])), 3)
    for sfx in ("", "_2"):
        v = g["v" + sfx]
        J, W = O.energy(v, m, model)
        assert J == g["J" + sfx]
        np.testing.assert_array_equal(W, g["densities" + sfx])
        np.testing.assert_array_equal(O.exact_gradient(v, m, p, model), g["g_exact" + sfx])
        np.testing.assert_array_equal(O.numeric_gradient(v, m, p, model, eps=1e-6),
                                      g["g_fd" + sfx])
    assert abs(g["J"] - 12.6623) < 5e-5                          # test_assembly.py:81-85
    assert np.isinf(O.energy(np.zeros(3 * m.nn), m, model)[0])
    with pytest.raises(O.OracleInadmissible):
        O.exact_gradient(np.zeros(3 * m.nn), m, p, model)
    with pytest.raises(O.OracleInadmissible, match=f"dof {int(g['fd_bad_dof_eps1'])}$"):
        O.numeric_gradient(m.nodes2coord.ravel().copy(), m, p, model, eps=1.0)


def test_bar_level2_bit_exact(golden):
    g = golden("bar2_mesh")
    m = O.bar_mesh(0.4, 0.01, 0.01, 2)
    np.testing.assert_array_equal(m.nodes2coord, g["coords"])
    np.testing.assert_array_equal(m.elems2nodes, g["conn"])
    np.testing.assert_array_equal(m.volumes, g["volumes"])
    np.testing.assert_array_equal(np.stack(m.dphi), g["dphi"])
    fixed = O.fixed_mask(m, [(lambda x: x[:, 0] < 1e-9, None),
                             (lambda x: x[:, 0] > 0.4 - 1e-9, None)], 3)
    m = O.mark_dirichlet(m, fixed, 3)
    np.testing.assert_array_equal(m.dofs_minim, g["dofs_minim"])
    p = O.build_patches(m)
    np.testing.assert_array_equal(p.lengths, g["p_lengths"])
    np.testing.assert_array_equal(p.elems, g["p_elems"])
    np.testing.assert_array_equal(p.slot, g["p_slot"])


def test_rect_problem_bit_exact(golden):
    g = golden("rect32x16_nh")
    m, model, b, v = O.problem_rect(32, 16, seed=2109)
    _check_mesh(m, g)
    p = O.build_patches(m)
    _check_patches(p, g)
    np.testing.assert_array_equal(v, g["v"])
    np.testing.assert_array_equal(b, g["b"])
    assert (model.params.C1, model.params.D1) == (g["C1"], g["D1"])
    assert O.energy(v, m, model, b)[0] == g["J"]
    np.testing.assert_array_equal(O.exact_gradient(v, m, p, model, b), g["g_exact"])
    np.testing.assert_array_equal(O.numeric_gradient(v, m, p, model, b, 1e-8), g["g_fd"])


def test_beam_problem_bit_exact(golden):
    g = golden("beam8x4x4_nh")
    m, model, b, v = O.problem_beam(8, 4, 4, seed=2109)
    _check_mesh(m, g)
    p = O.build_patches(m)
    _check_patches(p, g)
    np.testing.assert_array_equal(v, g["v"])
    np.testing.assert_array_equal(b, g["b"])
    assert O.energy(v, m, model, b)[0] == g["J"]
    np.testing.assert_array_equal(O.exact_gradient(v, m, p, model, b), g["g_exact"])
    np.testing.assert_array_equal(O.numeric_gradient(v, m, p, model, b, 1e-8), g["g_fd"])


def test_descent_loop_bit_exact(golden):
    """The config-5 first-order loop driven by the reference's energy and
    exact_gradient (tests/golden/make_golden.py case_descent)."""
    g = golden("descent_beam8x4x4")
    m, model, b, v = O.problem_beam(8, 4, 4, seed=2109)
    np.testing.assert_array_equal(v, g["v0"])
    p = O.build_patches(m)
    alpha = 1e-3 * (2.0 / 8) / np.abs(O.exact_gradient(v, m, p, model, b)).max()
    assert alpha == g["alpha"]
    Js, vf, gl = O.descent_loop(v, m, p, model, b, alpha, int(g["iters"]))
    np.testing.assert_array_equal(Js, g["J_hist"])
    np.testing.assert_array_equal(vf, g["v_final"])
    np.testing.assert_array_equal(gl, g["g_last"])
    assert (np.diff(Js) < 0).all()  # a descent loop: J decreases


def test_direct_fd_within_roundoff_of_reference_fd(golden):
    """The direct-sum FD (the GPU's summation structure) differs from the
    reference cumsum FD only by roundoff; both sit near the exact gradient."""
    for name, eps in (("cfg1_lshape4_p3", 1e-6), ("beam8x4x4_nh", 1e-8), ("rect32x16_nh", 1e-8)):
        g = golden(name)
        m = _mesh_from_golden(g)
        p = _patches_from_golden(g)
        if "C1" in g:
            model = O.Model("nh", O.LameParams(float(g["C1"]), float(g["D1"])), m.dim)
        else:
            model = O.Model("plap", O.PParams(float(g["p"])), 2)
        gd, scale = O.numeric_gradient_direct(g["v"], m, p, model, g["b"], eps)
        ref = g["g_fd"]
        gmax = np.abs(g["g_exact"]).max()
        # reference FD carries cumsum noise ~ u*|running sum|/eps; direct-sum
        # FD stays within that of the exact gradient
        assert np.abs(gd - g["g_exact"]).max() / gmax < 1e-4
        assert np.abs(gd - ref).max() / gmax < 1e-4


def test_density_known_answers():
    # test_models.py:78-83: W(2I) = C1 (9 - 6 log 2) + 49 D1
    prm = O.LameParams.from_E_nu_bulk(5.2, 0.3)
    F = [[np.array([2.0 if j == m else 0.0]) for m in range(3)] for j in range(3)]
    assert O.nh_W(F, prm)[0] == pytest.approx(prm.C1 * (9 - 6 * np.log(2)) + 49 * prm.D1,
                                              rel=1e-12)
    # test_models.py:131-136: p-Laplace (3,4), p=3 -> 125/3
    assert O.plap_W([[np.array([3.0]), np.array([4.0])]], O.PParams(3.0))[0] == \
        pytest.approx(125.0 / 3.0)
    # subgradient 0 at g = 0 for p < 2 (test_models.py:139-143)
    z = O.plap_dW([[np.zeros(2), np.zeros(2)]], O.PParams(1.5))
    assert (z[0][0] == 0).all() and (z[0][1] == 0).all()


def test_splitmix_reference_values():
    # fixed vectors of the shared counter-based generator (CUDA side must match)
    u = O.uniform01(2109, np.arange(4))
    assert u.dtype == np.float64 and ((0 <= u) & (u < 1)).all()
    assert O.splitmix64(np.array([0], dtype=np.uint64))[0] == np.uint64(0xE220A8397B1DCDAF)


def test_sampled_exact_gradient_matches_full(golden):
    """The per-dof restatement used for the full-size GPU checks agrees with the
    reference's exact gradient (golden) up to the cumsum roundoff."""
    g = golden("beam8x4x4_nh")
    m, model, b, v = O.problem_beam(8, 4, 4, seed=2109)
    p = O.build_patches(m)
    sample = np.arange(0, m.dofs_minim.size, 3)
    gs = O.sampled_exact_gradient(v, m.elems2nodes, m.volumes, m.dphi, p.prefix, p.elems, p.slot,
                                  m.nodes_minim, 3, model, b, m.dofs_minim, sample)
    ref = g["g_exact"][sample]
    assert np.abs(gs - ref).max() <= 1e-12 * np.abs(g["g_exact"]).max()


def _model_of(g, prefix=""):
    if prefix == "" and "C1" in g:
        return O.Model("nh", O.LameParams(float(g["C1"]), float(g["D1"])),
                       int(g["coords"].shape[1]))
    return None


def test_hole_mesh_unstructured_bit_exact(golden):
    """The reference's unstructured hole mesh (mesh.py:246-286): the oracle's
    partitions / patches / P1 data and evaluation reproduce it bit for bit."""
    g = golden("hole2")
    m = _mesh_from_golden(g)
    vol, dphi = O.p1_gradients(g["coords"], g["conn"])
    np.testing.assert_array_equal(vol, g["volumes"])
    np.testing.assert_array_equal(np.stack(dphi), g["dphi"])
    p = O.build_patches(m)
    _check_patches(p, g)
    model = _model_of(g)
    J, W = O.energy(g["v"], m, model, g["b"])
    assert J == g["J"]
    np.testing.assert_array_equal(W, g["densities"])
    np.testing.assert_array_equal(O.exact_gradient(g["v"], m, p, model, g["b"]), g["g_exact"])
    np.testing.assert_array_equal(O.numeric_gradient(g["v"], m, p, model, g["b"], 1e-8),
                                  g["g_fd"])
    gl = {k[3:]: val for k, val in g.items() if k.startswith("pl_")}
    m1 = _mesh_from_golden(gl)
    p1 = O.build_patches(m1)
    np.testing.assert_array_equal(p1.elems, gl["p_elems"])
    for pexp in (3.0, 1.8):
        pre = f"pl{pexp:g}_"
        model1 = O.Model("plap", O.PParams(pexp), 2)
        assert O.energy(g[pre + "v"], m1, model1, g[pre + "b"])[0] == g[pre + "J"]
        np.testing.assert_array_equal(O.exact_gradient(g[pre + "v"], m1, p1, model1, g[pre + "b"]),
                                      g[pre + "g_exact"])


def test_renumbered_beam_bit_exact(golden):
    """Generic numbering (nodes / elements permuted, vertices rotated)."""
    g = golden("beam6x3x3_renumbered")
    m = _mesh_from_golden(g)
    vol, dphi = O.p1_gradients(g["coords"], g["conn"])
    np.testing.assert_array_equal(vol, g["volumes"])
    np.testing.assert_array_equal(np.stack(dphi), g["dphi"])
    fixed = O.fixed_mask(m, [(O.left_face, None)], 3)
    mm = O.mark_dirichlet(m, fixed, 3)
    _check_mesh(mm, g)
    p = O.build_patches(mm)
    _check_patches(p, g)
    model = _model_of(g)
    assert O.energy(g["v"], mm, model, g["b"])[0] == g["J"]
    np.testing.assert_array_equal(O.exact_gradient(g["v"], mm, p, model, g["b"]), g["g_exact"])
    np.testing.assert_array_equal(O.numeric_gradient(g["v"], mm, p, model, g["b"], 1e-8),
                                  g["g_fd"])


def test_standalone_helpers_bit_exact(golden):
    """gather / evaluate_F / segment sums / nodal load / mass matrix /
    linear term of the reference (assembly.py:27-91, patches.py:74-83)."""
    g = golden("exports")
    for tag, d in (("l", 1), ("b", 3)):
        conn, V = g[f"{tag}_conn"], g[f"{tag}_V"]
        vals = O.element_values(V.ravel(), d, conn)
        np.testing.assert_array_equal(np.stack(vals), g[f"{tag}_gather"])
        F = O.grad_field(list(g[f"{tag}_dphi"]), vals)
        np.testing.assert_array_equal(np.array(F), g[f"{tag}_F"])
        np.testing.assert_array_equal(O.cumsum_segments(g[f"{tag}_rows"], g[f"{tag}_indx"]),
                                      g[f"{tag}_segsum"])
        m = O.OMesh(int(g[f"{tag}_coords"].shape[1]), -1, g[f"{tag}_coords"], conn,
                    g[f"{tag}_volumes"], list(g[f"{tag}_dphi"]), d, None, None, None, None,
                    None)
        M = O.mass_matrix(m)
        np.testing.assert_array_equal(M.indptr, g[f"{tag}_M_indptr"])
        np.testing.assert_array_equal(M.indices, g[f"{tag}_M_indices"])
        np.testing.assert_array_equal(M.data, g[f"{tag}_M_data"])
        np.testing.assert_array_equal(O.load_vector(m, g[f"{tag}_f_nodal"], d),
                                      g[f"{tag}_b_nodal"])
        assert float(g[f"{tag}_b_nodal"] @ g[f"{tag}_v"]) == g[f"{tag}_linear_term"]


def test_degenerate_decisions_match_reference(golden):
    """det F exactly at 0 (flattened element): +inf energy and the exact
    path's raise decided by the six-term determinant, as the reference."""
    g = golden("degenerate_beam4x2x2")
    m = _mesh_from_golden(g)
    p = _patches_from_golden(g)
    model = _model_of(g)
    for v, J, r in zip(g["v"], g["J"], g["raises"]):
        assert O.energy(v, m, model)[0] == J
        if r:
            with pytest.raises(O.OracleInadmissible):
                O.exact_gradient(v, m, p, model)
        else:
            O.exact_gradient(v, m, p, model)


def test_femmin_work_variant_bit_exact(golden):
    """The reference-arm variant (the reference's per-call work, patch-row
    copies and boolean owner mask) gives the reference's exact gradient."""
    for name in ("beam8x4x4_nh", "cfg1_lshape4_p3"):
        g = golden(name)
        m = _mesh_from_golden(g)
        p = _patches_from_golden(g)
        rp = O.reference_patches(m, p)
        if "C1" in g:
            model = O.Model("nh", O.LameParams(float(g["C1"]), float(g["D1"])), m.dim)
        else:
            model = O.Model("plap", O.PParams(float(g["p"])), 2)
        np.testing.assert_array_equal(O.exact_gradient_femmin(g["v"], m, rp, model, g["b"]),
                                      g["g_exact"])
