"""GPU tests of the SURVEY §8f rows beyond the minimizers: the Hessian
utilities (solver.py:344-398) against the reference's own outputs
(tests/golden/hessian.npz) and the device-side VTK writer."""

import numpy as np
import pytest

from oracle import femmin_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2109_01158_b200 as fb  # noqa: E402
from paper_2109_01158_b200 import hessian, problems, vtk_io  # noqa: E402


def _lshape1(golden):
    g = golden("lshape1_plap")
    m = fb.Mesh(dim=2, level=-1, nodes2coord=g["coords"], elems2nodes=g["conn"],
                volumes=g["volumes"], dphi=list(g["dphi"]), d=1,
                nodes_dirichlet=g["nodes_dirichlet"], nodes_minim=g["nodes_minim"],
                dofs_dirichlet=g["dofs_dirichlet"], dofs_minim=g["dofs_minim"],
                dofs_minim_local=g["dofs_minim_local"])
    return m, g


def _check_colors(indptr, indices, colors):
    for i in range(indptr.size - 1):
        cc = colors[indices[indptr[i]:indptr[i + 1]]]
        assert len(set(cc.tolist())) == cc.size


def test_pattern_bit_exact_and_coloring(golden):
    h = golden("hessian")
    m, _ = _lshape1(golden)
    P = fb.hessian_sparsity(m, 1)
    np.testing.assert_array_equal(P.indptr, h["l_indptr"])
    np.testing.assert_array_equal(P.indices, h["l_indices"])
    assert (P != P.T).nnz == 0
    _check_colors(P.indptr, P.indices, fb.greedy_coloring(P))
    pr = problems.beam(8, 4, 4, seed=2109, keep=True)
    ip, ix = hessian.hessian_pattern_device(pr.meta["conn"], pr.nn, 3, pr.meta["dofs_minim"])
    np.testing.assert_array_equal(ip.cpu().numpy(), h["b_indptr"])
    np.testing.assert_array_equal(ix.cpu().numpy(), h["b_indices"])
    cols, nc = hessian.color_device(ip, ix)
    _check_colors(h["b_indptr"], h["b_indices"], cols.cpu().numpy())
    assert nc == int(cols.max()) + 1


def test_fd_hessian_plaplace_p2_is_stiffness(golden):
    """The reference test (test_solver.py:161-185): the coloured FD Hessian
    of the p = 2 energy is the stiffness matrix (atol 1e-5); and it matches
    the reference's own coloured FD Hessian."""
    h = golden("hessian")
    m, g = _lshape1(golden)
    P = fb.Patches(lengths=g["p_lengths"], elems=g["p_elems"], volumes=None, elems2nodes=None,
                   dphi=None, logical=None, prefix=g["p_prefix"], slot=g["p_slot"])
    model = fb.PLaplacian(fb.PLaplaceParams(p=2.0), dim=2)
    load = fb.LinearLoad.assemble(m, -10.0, d=1)
    dm = fb.context_for(m, P, d=1)
    v = torch.zeros(m.nn, dtype=torch.float64, device="cuda")
    b = torch.as_tensor(load.b).cuda()
    ip, ix, vals, nc = hessian.fd_hessian_device(dm, v, model, b, m.elems2nodes, m.dofs_minim)
    H = hessian._to_scipy(ip, ix, ip.numel() - 1, vals.cpu().numpy()).toarray()
    np.testing.assert_allclose(H, h["l_K"], atol=1e-5)
    np.testing.assert_allclose(H, h["l_H"], rtol=0, atol=1e-6 * np.abs(h["l_H"]).max())
    # the host-callable drop-in on the same problem
    def gx(x):
        vv = np.zeros(m.nn)
        vv[m.dofs_minim] = x
        return fb.exact_gradient(vv, m, P, model, load)
    H2 = fb.colored_fd_hessian(gx, np.zeros(m.dofs_minim.size), fb.hessian_sparsity(m, 1))
    np.testing.assert_allclose(H2.toarray(), h["l_H"], rtol=0, atol=1e-6 * np.abs(h["l_H"]).max())


def test_fd_hessian_neo_hookean_vs_reference(golden):
    """8x4x4 config-4 beam at the seeded field: the device coloured FD Hessian
    against the reference's; with the reference's own (greedy) colours the
    device result is bit-identical to the one with the device colours."""
    h = golden("hessian")
    pr = problems.beam(8, 4, 4, seed=2109, keep=True)
    assert np.array_equal(pr.v.cpu().numpy(), h["b_v"])
    om, omodel, b, _ = O.problem_beam(8, 4, 4, seed=2109)
    bd = torch.from_numpy(b).cuda()
    conn, dmin = pr.meta["conn"], pr.meta["dofs_minim"]
    ip, ix, vals, nc = hessian.fd_hessian_device(pr.dm, pr.v, pr.model, bd, conn, dmin)
    ref = np.zeros(ix.numel())
    Href = hessian._to_scipy(torch.from_numpy(h["b_H_indptr"]), torch.from_numpy(h["b_H_indices"]),
                             600, h["b_H_data"]).toarray()
    H = hessian._to_scipy(ip, ix, 600, vals.cpu().numpy()).toarray()
    scale = np.abs(Href).max()
    # both are forward differences with step 1e-6 of gradients that agree to
    # ~1e-14 relative: |dH| ~ 1e-14 |g| / 1e-6
    assert np.abs(H - Href).max() <= 1e-6 * scale, np.abs(H - Href).max() / scale
    _, _, vals2, _ = hessian.fd_hessian_device(pr.dm, pr.v, pr.model, bd, conn, dmin,
                                               colors=h["b_colors"], pattern=(ip, ix))
    assert torch.equal(vals, vals2)
    del ref


def test_solution_vtk_from_device(tmp_path):
    pr = problems.beam(8, 4, 4, seed=2109, keep=True)
    om, omodel, b, v = O.problem_beam(8, 4, 4, seed=2109)
    path = tmp_path / "sol.vtk"
    vtk_io.write_solution_vtk(path, pr.meta["coords"], pr.meta["conn"], pr.v, 3, model=pr.model,
                              dm=pr.dm, b=pr.b)
    pts, cells, pdata, cdata = vtk_io.read_vtk(path)
    np.testing.assert_array_equal(pts, v.reshape(-1, 3))
    np.testing.assert_array_equal(cells, om.elems2nodes)
    W = O.energy(v, om, omodel, b)[1]
    np.testing.assert_allclose(cdata["density"], W, rtol=1e-13)


def _embed(n_full, dofs, x):
    p = torch.zeros(n_full, dtype=torch.float64, device="cuda")
    p[torch.as_tensor(dofs, device="cuda")] = x
    return p


def test_exact_hvp_p2_is_stiffness(golden):
    """fm_hvp_exact for p = 2 is the P1 stiffness matrix (the reference's
    bench.assemble_stiffness_matrix, restricted to the free dofs)."""
    h = golden("hessian")
    m, g = _lshape1(golden)
    P = fb.Patches(lengths=g["p_lengths"], elems=g["p_elems"], volumes=None, elems2nodes=None,
                   dphi=None, logical=None, prefix=g["p_prefix"], slot=g["p_slot"])
    model = fb.PLaplacian(fb.PLaplaceParams(p=2.0), dim=2)
    dm = fb.context_for(m, P, d=1)
    rng = np.random.default_rng(3)
    v = torch.as_tensor(rng.normal(size=m.nn)).cuda()
    x = rng.normal(size=m.dofs_minim.size)
    hp = dm.hvp(v, _embed(m.nn, m.dofs_minim, torch.as_tensor(x).cuda()), model)
    dm.check()
    ref = h["l_K"] @ x
    assert np.abs(hp.cpu().numpy() - ref).max() <= 1e-13 * np.abs(ref).max()


@pytest.mark.parametrize("kind", ["beam", "lshape_p3", "lshape_p18", "rect"])
def test_exact_hvp_vs_gradient_differences(kind):
    """H p against central differences of the exact gradient (h = 1e-6 |v|/|p|:
    truncation + roundoff ~1e-8 of |Hp|) and symmetry q.Hp = p.Hq."""
    if kind == "beam":
        pr = problems.beam(16, 8, 8, seed=4)
    elif kind == "rect":
        pr = problems.rect(64, 32, seed=4)
    else:
        pr = problems.lshape(5, 3.0 if kind == "lshape_p3" else 1.8, seed=4, keep=True)
    dm, model = pr.dm, pr.model
    dofs = (pr.meta["dofs_minim"] if "dofs_minim" in pr.meta else None)
    gen = torch.Generator(device="cuda").manual_seed(5)
    nf = dm.nfree_dofs
    xp = torch.rand(nf, generator=gen, device="cuda", dtype=torch.float64) - 0.5
    xq = torch.rand(nf, generator=gen, device="cuda", dtype=torch.float64) - 0.5
    p, q = _embed(pr.v.numel(), dofs, xp), _embed(pr.v.numel(), dofs, xq)
    hp = dm.hvp(pr.v, p, model)
    hq = dm.hvp(pr.v, q, model)
    dm.check()
    h = 1e-6 * float(pr.v.abs().max()) / float(p.abs().max())
    fd = (dm.exact_gradient(pr.v + h * p, model, pr.b) -
          dm.exact_gradient(pr.v - h * p, model, pr.b)) / (2 * h)
    scale = float(hp.abs().max())
    assert float((hp - fd).abs().max()) <= 2e-6 * scale, float((hp - fd).abs().max()) / scale
    a, b_ = float(torch.dot(xq, hp)), float(torch.dot(xp, hq))
    assert abs(a - b_) <= 1e-12 * max(abs(a), abs(b_), 1e-300)


def test_exact_hvp_matches_reference_fd_hessian(golden):
    """8x4x4 beam at the seeded field: H p against the reference's coloured FD
    Hessian times p (its own FD noise level, 1e-6 of the scale)."""
    h = golden("hessian")
    pr = problems.beam(8, 4, 4, seed=2109, keep=True)
    Href = hessian._to_scipy(torch.from_numpy(h["b_H_indptr"]), torch.from_numpy(h["b_H_indices"]),
                             600, h["b_H_data"])
    x = np.random.default_rng(9).normal(size=600)
    hp = pr.dm.hvp(pr.v, _embed(pr.v.numel(), pr.meta["dofs_minim"], torch.as_tensor(x).cuda()),
                   pr.model)
    ref = Href @ x
    assert np.abs(hp.cpu().numpy() - ref).max() <= 1e-6 * np.abs(ref).max()


def test_reports_bench1_3_on_gpu(tmp_path):
    """The reference's hot-path benchmarks 1-3 as CSV reports on the engine
    (reports.py; bench.py:208-296): counts of test_reports_io.py, the twisted
    bar's J at level 1 (test_acceptance.py:66) and exact-vs-FD agreement."""
    from paper_2109_01158_b200 import reports
    r1 = reports.bench1([1])
    c = {k: i for i, k in enumerate(r1.columns)}
    row = r1.rows[0]
    assert (row[c["nodes"]], row[c["elements"]], row[c["free_dofs"]],
            row[c["patch_rows"]]) == (729, 1920, 2133, 7584)
    r2 = reports.bench2([1], repeats=1)
    assert abs(r2.column("J_grad")[0] - 12.6623) < 5e-5
    r3 = reports.bench3([1], repeats=1)
    assert r3.column("rel_agreement")[0] < 1e-4
    path = tmp_path / "b3.csv"
    r3.to_csv(path)
    assert reports.BenchmarkReport.from_csv("bench3", path).rows == r3.rows
