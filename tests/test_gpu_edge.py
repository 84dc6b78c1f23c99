"""Edge cases of the path on the GPU, against the oracle / the reference's
behaviour: component-wise Dirichlet data (nodes with some components free:
the free-mask bits of the output offsets), a single element, a mesh without
free dofs, a free node without elements (PatchStructureError, patches.py:
57-59) and a flipped element (DegenerateElementError, mesh.py:92-96)."""

import numpy as np
import pytest

from oracle import femmin_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2109_01158_b200 as fb  # noqa: E402

J_TOL = G_TOL = 1e-10
FD_FACTOR = 64.0


def _fb_mesh(om):
    return fb.Mesh(dim=om.dim, level=-1, nodes2coord=om.nodes2coord, elems2nodes=om.elems2nodes,
                   volumes=om.volumes, dphi=list(om.dphi), d=om.d,
                   nodes_dirichlet=om.nodes_dirichlet, nodes_minim=om.nodes_minim,
                   dofs_dirichlet=om.dofs_dirichlet, dofs_minim=om.dofs_minim,
                   dofs_minim_local=om.dofs_minim_local)


def _nh(dim):
    prm = O.LameParams.from_E_nu_lambda(2e8, 0.3)
    return (fb.NeoHookean(fb.LameParams(prm.C1, prm.D1), dim=dim), O.Model("nh", prm, dim))


def _check_all(om, v, b, model, omodel, eps=1e-8):
    m = _fb_mesh(om)
    pt = fb.build_patches(m)
    op = O.build_patches(om)
    np.testing.assert_array_equal(pt.elems, op.elems)
    np.testing.assert_array_equal(pt.slot, op.slot)
    load = fb.LinearLoad(b=b)
    J, g = fb.energy_and_gradient(v, m, pt, model, load)
    Jo = O.energy(v, om, omodel, b)[0]
    go = O.exact_gradient(v, om, op, omodel, b)
    assert g.shape == go.shape
    assert abs(J - Jo) <= J_TOL * abs(Jo)
    if go.size:
        assert np.abs(g - go).max() <= G_TOL * np.abs(go).max()
        gn = fb.numeric_gradient(v, m, pt, model, load, eps=eps)
        gd, scale = O.numeric_gradient_direct(v, om, op, omodel, b, eps)
        assert (np.abs(gn - gd) <= FD_FACTOR * scale + 1e-300).all()
    return g


def test_componentwise_dirichlet():
    """x1 = 0 clamped, x1 = 2 only u_y fixed (a roller face): nodes with one
    or two free components; partitions bit-exact, evaluation vs the oracle."""
    om = O.beam_mesh(12, 6, 6, 0.0, 2.0, 0.0, 1.0, 0.0, 1.0)
    fixed = O.fixed_mask(om, [(O.left_face, None), (lambda x: x[:, 0] > 2.0 - 1e-9, [1]),
                              (lambda x: x[:, 2] < 1e-9, [0, 2])], 3)
    om = O.mark_dirichlet(om, fixed, 3)
    spec = fb.DirichletSpec([
        fb.DirichletRegion(where=lambda x: x[:, 0] < 1e-9),
        fb.DirichletRegion(where=lambda x: x[:, 0] > 2.0 - 1e-9, components=[1]),
        fb.DirichletRegion(where=lambda x: x[:, 2] < 1e-9, components=[0, 2])])
    raw = fb.Mesh(dim=3, level=-1, nodes2coord=om.nodes2coord, elems2nodes=om.elems2nodes,
                  volumes=om.volumes, dphi=list(om.dphi), d=3)
    mm = fb.mark_dirichlet(raw, spec, d=3)
    for k in ("nodes_dirichlet", "nodes_minim", "dofs_dirichlet", "dofs_minim",
              "dofs_minim_local"):
        np.testing.assert_array_equal(getattr(mm, k), getattr(om, k), err_msg=k)
    partial = np.unique(om.dofs_minim // 3, return_counts=True)[1]
    assert (partial < 3).any() and (partial == 3).any()  # mixed masks exercised
    model, omodel = _nh(3)
    v = O.field_nh(om, 19, 1e-2 * 2.0 / 12)
    b = O.load_vector(om, (0.0, 0.0, -2.5e7), 3)
    _check_all(om, v, b, model, omodel)


def test_single_element():
    """One tetrahedron, one free node."""
    coords = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]])
    conn = np.array([[0, 1, 2, 3]])
    om = O._assemble_mesh(3, -1, coords, conn)
    om = O.mark_dirichlet(om, O.fixed_mask(om, [(lambda x: x[:, 0] < 0.5, None)], 3), 3)
    assert om.nodes_minim.tolist() == [1]
    model, omodel = _nh(3)
    v = coords.ravel() * 1.01
    b = O.load_vector(om, (0.0, 0.0, -2.5e7), 3)
    g = _check_all(om, v, b, model, omodel)
    assert g.shape == (3,)


def test_no_free_dofs():
    """Every node clamped: J is still the energy; the gradients are empty."""
    om = O.beam_mesh(4, 2, 2, 0.0, 2.0, 0.0, 1.0, 0.0, 1.0)
    om = O.mark_dirichlet(om, O.fixed_mask(om, [(lambda x: x[:, 0] > -1.0, None)], 3), 3)
    assert om.dofs_minim.size == 0
    m = _fb_mesh(om)
    model, omodel = _nh(3)
    v = O.field_nh(om, 3, 0.0) * 1.001
    b = O.load_vector(om, (0.0, 0.0, -2.5e7), 3)
    J, W = fb.energy(v, m, model, fb.LinearLoad(b=b))
    assert abs(J - O.energy(v, om, omodel, b)[0]) <= J_TOL * abs(J)
    pt = fb.Patches(lengths=np.zeros(0, np.int64), elems=np.zeros(0, np.int64), volumes=None,
                    elems2nodes=None, dphi=None, logical=None, prefix=np.zeros(0, np.int64),
                    slot=np.zeros(0, np.int64))
    assert fb.exact_gradient(v, m, pt, model).shape == (0,)
    assert fb.numeric_gradient(v, m, pt, model).shape == (0,)


def test_free_node_without_elements():
    """patches.py:57-59: a free node that no element touches."""
    coords = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [5.0, 5.0]])
    conn = np.array([[0, 1, 2]])
    vol, dphi = fb.compute_p1_gradients(coords, conn)
    m = fb.Mesh(dim=2, level=-1, nodes2coord=coords, elems2nodes=conn, volumes=vol,
                dphi=dphi, d=1)
    m = fb.mark_dirichlet(m, fb.DirichletSpec([fb.DirichletRegion(
        where=lambda x: x[:, 0] + x[:, 1] < 0.5)]), d=1)
    with pytest.raises(fb.PatchStructureError, match="free node 3 has an empty patch"):
        fb.build_patches(m)
    assert issubclass(fb.PatchStructureError, ValueError)


def test_flipped_element():
    """mesh.py:92-96: the first element with a nonpositive measure."""
    coords = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [1.0, 1.0]])
    conn = np.array([[0, 1, 2], [1, 2, 3]])  # the second is clockwise
    with pytest.raises(fb.DegenerateElementError, match="element 1 has nonpositive measure"):
        fb.compute_p1_gradients(coords, conn)
    assert issubclass(fb.DegenerateElementError, ValueError)


@pytest.mark.parametrize("scale", [1e-4, 1e5])
def test_scaled_coordinates(scale):
    """Meshes far from unit size (the tile boxes derive from the mean element
    measure; det F is dimensionless): J and the gradients follow the oracle."""
    om = O.beam_mesh(10, 5, 5, 0.0, 2.0 * scale, 0.0, scale, 0.0, scale)
    om = O.mark_dirichlet(om, O.fixed_mask(om, [(lambda x: x[:, 0] < 1e-9 * scale, None)], 3), 3)
    model, omodel = _nh(3)
    v = O.field_nh(om, 23, 1e-2 * 0.2 * scale)
    b = O.load_vector(om, (0.0, 0.0, -2.5e7), 3)
    _check_all(om, v, b, model, omodel, eps=1e-8 * scale)


def test_componentwise_dirichlet_2d():
    """2D Neo-Hookean with x fixed on the left edge and y on the bottom edge."""
    om = O.rect_mesh(16, 8)
    om = O.mark_dirichlet(om, O.fixed_mask(om, [(lambda x: x[:, 0] < 1e-9, [0]),
                                                (lambda x: x[:, 1] < 1e-9, [1])], 2), 2)
    model, omodel = _nh(2)
    v = O.field_nh(om, 29, 1e-2 * 2.0 / 16)
    b = O.load_vector(om, (0.0, -3.5e7), 2)
    _check_all(om, v, b, model, omodel)


def test_concurrent_drop_in_calls():
    """The reference functions are pure: concurrent calls on one
    mesh from several threads, one of them on an inadmissible field, give the
    serial results and raise only in the offending thread."""
    import threading
    om = O.beam_mesh(12, 6, 6, 0.0, 2.0, 0.0, 1.0, 0.0, 1.0)
    om = O.mark_dirichlet(om, O.fixed_mask(om, [(O.left_face, None)], 3), 3)
    m = _fb_mesh(om)
    pt = fb.build_patches(m)
    model, _ = _nh(3)
    load = fb.LinearLoad(b=O.load_vector(om, (0.0, 0.0, -2.5e7), 3))
    fields = [O.field_nh(om, 100 + k, 1e-2 * 2.0 / 12) for k in range(6)]
    fields[3] = np.zeros_like(fields[3])  # inadmissible: det F = 0
    serial = []
    for k, v in enumerate(fields):
        try:
            serial.append(fb.energy_and_gradient(v, m, pt, model, load))
        except fb.InadmissibleStateError:
            serial.append("raise")
    assert serial[3] == "raise"
    out = [None] * len(fields)

    def work(k):
        for _ in range(5):
            try:
                out[k] = fb.energy_and_gradient(fields[k], m, pt, model, load)
            except fb.InadmissibleStateError:
                out[k] = "raise"
    threads = [threading.Thread(target=work, args=(k,)) for k in range(len(fields))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for a, b in zip(out, serial):
        if isinstance(b, str):
            assert a == b
        else:
            assert a[0] == b[0] and np.array_equal(a[1], b[1])
