"""Minimizers (reference solver.py).

CPU: the trust-region / L-BFGS core of paper_2109_01158_b200.solver driven by
the oracle's J and grad J on the reference's unit-test fixture
lshape_problem(1), against the reference minimizers' own results
(tests/golden/minimize_lshape1.npz, made by tests/golden/make_golden.py), plus
the reference's option / error behaviour.  GPU: the device-resident
``minimize_device`` on the same problem.
"""

import numpy as np
import pytest
import torch

from oracle import femmin_oracle as O
from paper_2109_01158_b200.solver import (InvalidStartError, SolveOptions, StagnationError,
                                          continuation_solve, minimize)


def _omesh(g):
    return O.OMesh(int(g["coords"].shape[1]), -1, g["coords"], g["conn"], g["volumes"],
                   list(g["dphi"]), int(g["d"]), g["nodes_dirichlet"], g["nodes_minim"],
                   g["dofs_dirichlet"], g["dofs_minim"], g["dofs_minim_local"])


def _oracle_problem(golden, p):
    g = golden("lshape1_plap")
    m = _omesh(g)
    P = O.build_patches(m)
    model = O.Model("plap", O.PParams(p), 2)
    b = golden("minimize_lshape1")["b"]

    def J(v):
        return O.energy(v, m, model, b)[0]

    def gr(v):
        return O.exact_gradient(v, m, P, model, b)

    return m, J, gr


def test_options_validation():
    with pytest.raises(ValueError):
        SolveOptions(tol_g=0.0)
    with pytest.raises(ValueError):
        SolveOptions(solver="newton")


def test_convex_quadratic_converges_fast():
    n = 12
    res = minimize(lambda v: 0.5 * float(v @ v), lambda v: v.copy(), np.ones(n), np.arange(n))
    assert res.converged and res.iters <= 5
    assert abs(res.J_u) < 1e-12 and np.abs(res.u).max() < 1e-6


@pytest.mark.parametrize("p", [3.0, 2.0])
def test_trust_region_matches_reference(golden, p):
    ref = golden("minimize_lshape1")
    m, J, gr = _oracle_problem(golden, p)
    res = minimize(J, gr, np.zeros(m.nodes2coord.shape[0]), m.dofs_minim, SolveOptions())
    tag = f"p{p:g}"
    assert res.converged and res.status == str(ref[f"tr_status_{tag}"])
    assert res.iters == int(ref[f"tr_iters_{tag}"])
    assert abs(res.J_u - float(ref[f"tr_J_{tag}"])) <= 1e-12 * abs(float(ref[f"tr_J_{tag}"]))
    np.testing.assert_allclose(res.u, ref[f"tr_u_{tag}"], rtol=0, atol=1e-9)
    if p == 2.0:  # the quadratic case agrees with the direct Poisson solve
        assert res.J_u == pytest.approx(float(ref["direct_J_p2"]), rel=1e-8)


def test_lbfgs_matches_reference(golden):
    ref = golden("minimize_lshape1")
    m, J, gr = _oracle_problem(golden, 3.0)
    res = minimize(J, gr, np.zeros(m.nodes2coord.shape[0]), m.dofs_minim,
                   SolveOptions(solver="lbfgs", tol_g=1e-8, tol_f=1e-12, tol_step=1e-8))
    assert res.J_u == pytest.approx(float(ref["lbfgs_J_p3"]), abs=1e-10)
    assert res.J_u == pytest.approx(float(ref["tr_J_p3"]), abs=1e-5)


def test_dirichlet_entries_preserved_and_errors(golden):
    m, J, gr = _oracle_problem(golden, 3.0)
    v0 = np.zeros(m.nodes2coord.shape[0])
    v0[m.dofs_dirichlet] = 0.125
    res = minimize(J, gr, v0, m.dofs_minim)
    assert (res.u[m.dofs_dirichlet] == 0.125).all()
    with pytest.raises(InvalidStartError):
        minimize(lambda v: float("inf"), gr, v0, m.dofs_minim)
    with pytest.raises(InvalidStartError, match="load step 1"):
        continuation_solve(lambda v: float("inf"), gr, v0, m.dofs_minim, m.dofs_dirichlet,
                           [np.zeros(m.dofs_dirichlet.size)])


def test_continuation_warm_start(golden):
    m, J, gr = _oracle_problem(golden, 3.0)
    bnd = m.dofs_dirichlet
    sched = [0.05 * t * np.ones(bnd.size) for t in range(1, 4)]
    seen = []
    res = continuation_solve(J, gr, np.zeros(m.nodes2coord.shape[0]), m.dofs_minim, bnd, sched,
                             callback=lambda t, r: seen.append(t))
    assert seen == [1, 2, 3]
    for bc, r in zip(sched, res):
        np.testing.assert_array_equal(r.u[bnd], bc)
        assert r.converged


def test_stagnation_error():
    # a function whose model never predicts a decrease: |g| stays, H negative
    # curvature along g is unbounded -> radius shrinks to nothing eventually
    n = 3
    with pytest.raises(StagnationError):
        minimize(lambda v: float(v[0]) if v[0] > -1e-300 else float("inf"),
                 lambda v: np.array([1.0, 0.0, 0.0]), np.zeros(n), np.arange(n),
                 SolveOptions(max_iters=10000, tr_radius0=1e-10))


@pytest.mark.gpu
@pytest.mark.parametrize("hvp", ["fd", "exact"])
@pytest.mark.parametrize("p", [3.0, 2.0])
def test_minimize_device_matches_reference(golden, p, hvp):
    import paper_2109_01158_b200 as fb
    from paper_2109_01158_b200.solver import minimize_device
    g = golden("lshape1_plap")
    ref = golden("minimize_lshape1")
    m = fb.Mesh(dim=2, level=-1, nodes2coord=g["coords"], elems2nodes=g["conn"],
                volumes=g["volumes"], dphi=list(g["dphi"]), d=1,
                nodes_dirichlet=g["nodes_dirichlet"], nodes_minim=g["nodes_minim"],
                dofs_dirichlet=g["dofs_dirichlet"], dofs_minim=g["dofs_minim"],
                dofs_minim_local=g["dofs_minim_local"])
    dm = fb.context_for(m)
    model = fb.PLaplacian(fb.PLaplaceParams(p=p), dim=2)
    b = torch.from_numpy(ref["b"]).cuda()
    v0 = torch.zeros(m.nn, dtype=torch.float64, device="cuda")
    dofs = torch.from_numpy(np.asarray(m.dofs_minim)).cuda()
    res = minimize_device(dm, model, b, v0, dofs, SolveOptions(hvp=hvp))
    tag = f"p{p:g}"
    # (the exact Hessian-vector product changes the CG iterates, not the minimizer)
    assert res.converged
    if hvp == "fd":
        assert res.status == str(ref[f"tr_status_{tag}"])
    else:
        assert res.n_hvp > 0
    assert res.J_u == pytest.approx(float(ref[f"tr_J_{tag}"]), rel=1e-10)
    np.testing.assert_allclose(res.u.cpu().numpy(), ref[f"tr_u_{tag}"], rtol=0, atol=1e-7)
    assert (res.u[dofs.new_tensor(np.asarray(m.dofs_dirichlet))] == 0).all()


@pytest.mark.gpu
@pytest.mark.parametrize("hvp", ["fd", "exact"])
def test_minimize_device_beam_decreases_energy(hvp):
    """A Neo-Hookean beam under load: the device trust region converges from
    the reference configuration and every accepted step lowers J."""
    from paper_2109_01158_b200 import problems
    from paper_2109_01158_b200.solver import minimize_device
    pr = problems.beam(8, 4, 4, seed=1)
    v0 = pr.v.clone()
    J0 = float(pr.dm.energy(v0, pr.model, pr.b)[0])
    res = minimize_device(pr.dm, pr.model, pr.b, v0, pr.meta["dofs_minim"],
                          SolveOptions(tol_g=1e-7, max_iters=200, hvp=hvp))
    assert res.converged and res.J_u < J0
    g = pr.dm.exact_gradient(res.u, pr.model, pr.b)
    g0 = pr.dm.exact_gradient(v0, pr.model, pr.b)
    assert float(g.abs().max()) <= 1e-7 * max(1.0, float(g0.abs().max())) * 1.0001


@pytest.mark.gpu
@pytest.mark.parametrize("hvp", ["fd", "exact"])
def test_device_cg_matches_host_cg(golden, hvp):
    """The device-resident CG (csrc/fm_cg.cu) takes the host loop's iterates:
    same outer iterations, status and gradient-call count, J to 1e-12."""
    import paper_2109_01158_b200 as fb
    from paper_2109_01158_b200.solver import minimize_device
    g = golden("lshape1_plap")
    ref = golden("minimize_lshape1")
    m = fb.Mesh(dim=2, level=-1, nodes2coord=g["coords"], elems2nodes=g["conn"],
                volumes=g["volumes"], dphi=list(g["dphi"]), d=1,
                nodes_dirichlet=g["nodes_dirichlet"], nodes_minim=g["nodes_minim"],
                dofs_dirichlet=g["dofs_dirichlet"], dofs_minim=g["dofs_minim"],
                dofs_minim_local=g["dofs_minim_local"])
    dm = fb.context_for(m)
    model = fb.PLaplacian(fb.PLaplaceParams(p=3.0), dim=2)
    b = torch.from_numpy(ref["b"]).cuda()
    v0 = torch.zeros(m.nn, dtype=torch.float64, device="cuda")
    dofs = torch.from_numpy(np.asarray(m.dofs_minim)).cuda()
    a = minimize_device(dm, model, b, v0, dofs, SolveOptions(hvp=hvp, device_cg=True))
    h = minimize_device(dm, model, b, v0, dofs, SolveOptions(hvp=hvp, device_cg=False))
    assert a.converged and h.converged and a.status == h.status
    assert a.iters == h.iters and a.n_grad == h.n_grad
    assert abs(a.J_u - h.J_u) <= 1e-12 * abs(h.J_u)
    assert float((a.u - h.u).abs().max()) <= 1e-9
