"""Generate the golden vectors of tests/golden/*.npz from the REAL reference.

Run in the build container (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every output array below is produced by the unmodified reference package
``femmin`` (/root/reference/pkg/src/femmin).  Inputs (trial fields) come from
the counter-based generator in ``oracle/femmin_oracle.py`` or from the
reference test seeds; the meshes the reference cannot build (config-3
rectangle, config-4/5 beam) are composed from reference pieces
(``_grid_triangles``, ``_make_mesh``, ``mark_dirichlet``) exactly as
SURVEY.md §0.1 #3/#4 describes.  The fixtures are small (a few MB in total).
"""

import os
import re
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import femmin  # noqa: E402
from femmin import bench, mesh as fmesh, patches as fpatches  # noqa: E402
from femmin.assembly import LinearLoad, energy, interpolate  # noqa: E402
from femmin.gradients import exact_gradient, numeric_gradient  # noqa: E402
from femmin.models import (ElasticParams, InadmissibleStateError, NeoHookean,  # noqa: E402
                           PLaplaceParams, PLaplacian)

from oracle import femmin_oracle as O  # noqa: E402  (inputs only)


class Lame:
    def __init__(self, C1, D1):
        self.C1, self.D1 = C1, D1


def _mesh_arrays(m):
    return dict(
        coords=m.nodes2coord, conn=m.elems2nodes, volumes=m.volumes,
        dphi=np.stack(m.dphi), d=np.int64(m.d),
        nodes_dirichlet=m.nodes_dirichlet, nodes_minim=m.nodes_minim,
        dofs_dirichlet=m.dofs_dirichlet, dofs_minim=m.dofs_minim,
        dofs_minim_local=m.dofs_minim_local)


def _patch_arrays(p):
    return dict(p_lengths=p.lengths, p_prefix=p.prefix, p_elems=p.elems,
                p_slot=np.argmax(p.logical, axis=1).astype(np.int64),
                p_indx3=fpatches.patch_prefix_indices(p, 3))


def _evaluate(m, p, model, load, v, fd_eps):
    J, W = energy(v, m, model, load)
    ge = exact_gradient(v, m, p, model, load)
    gn = numeric_gradient(v, m, p, model, load, eps=fd_eps)
    return dict(v=v, J=np.float64(J), densities=W, g_exact=ge, g_fd=gn,
                fd_eps=np.float64(fd_eps),
                b=(load.b if load is not None else np.zeros(m.d * m.nn)))


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"{name}: {os.path.getsize(path) / 1e3:.0f} kB")


def case_lshape(level, p, seed, name, fd_eps=1e-6):
    m = bench.lshape_problem(level)
    pt = femmin.build_patches(m)
    model = PLaplacian(PLaplaceParams(p=p), dim=2)
    load = LinearLoad.assemble(m, -10.0, d=1)
    v = np.zeros(m.nn)
    v[m.dofs_minim] = O.uniform01(seed, m.dofs_minim)
    save(name, **_mesh_arrays(m), **_patch_arrays(pt),
         **_evaluate(m, pt, model, load, v, fd_eps), p=np.float64(p),
         level=np.int64(level), seed=np.int64(seed))


def case_bar_twist():
    m = bench.bar_problem(1)
    pt = femmin.build_patches(m)
    model = NeoHookean(bench.BAR_MATERIAL, dim=3)
    v = interpolate(bench.twist_map(2 * np.pi), m, d=3)
    out = _evaluate(m, pt, model, None, v, 1e-6)
    # admissible random affine field + noise, as test_gradients.py:21-28
    rng = np.random.default_rng(20240817)
    A = np.eye(3) + 0.05 * rng.normal(size=(3, 3))
    while np.linalg.det(A) < 0.5:
        A = np.eye(3) + 0.05 * rng.normal(size=(3, 3))
    v2 = interpolate(lambda x: x @ A.T, m, d=3) + 1e-6 * rng.normal(size=3 * m.nn)
    out2 = _evaluate(m, pt, model, None, v2, 1e-6)
    # inadmissible behaviour: collapsed field and a huge FD step at identity
    J0, W0 = energy(np.zeros(3 * m.nn), m, model)
    try:
        numeric_gradient(interpolate(lambda x: x, m, d=3), m, pt, model, eps=1.0)
        bad_dof = -1
    except InadmissibleStateError as exc:
        bad_dof = int(re.search(r"dof (\d+)", str(exc)).group(1))
    save("bar1_nh", **_mesh_arrays(m), **_patch_arrays(pt), **out,
         **{k + "_2": val for k, val in out2.items()},
         C1=np.float64(bench.BAR_MATERIAL.C1), D1=np.float64(bench.BAR_MATERIAL.D1),
         J_collapsed=np.float64(J0), fd_bad_dof_eps1=np.int64(bad_dof))


def case_bar2_mesh():
    m = bench.bar_problem(2)
    pt = femmin.build_patches(m)
    save("bar2_mesh", coords=m.nodes2coord, conn=m.elems2nodes, volumes=m.volumes,
         dphi=np.stack(m.dphi), nodes_minim=m.nodes_minim, dofs_minim=m.dofs_minim,
         p_lengths=pt.lengths, p_elems=pt.elems,
         p_slot=np.argmax(pt.logical, axis=1).astype(np.int64))


def case_rect(nx, ny, seed):
    xs = np.linspace(0.0, 2.0, nx + 1)
    ys = np.linspace(0.0, 1.0, ny + 1)
    Y, X = np.meshgrid(ys, xs, indexing="ij")
    coords = np.column_stack([X.ravel(), Y.ravel()])
    tri, _, _ = fmesh._grid_triangles(nx, ny)
    m = fmesh._make_mesh(2, -1, coords, tri)
    spec = fmesh.DirichletSpec([fmesh.DirichletRegion(where=lambda x: x[:, 0] < 1e-9)])
    m = fmesh.mark_dirichlet(m, spec, d=2)
    pt = femmin.build_patches(m)
    E, nu = 2e8, 0.3
    mu, lam = E / (2 * (1 + nu)), E * nu / ((1 + nu) * (1 - 2 * nu))
    model = NeoHookean(ElasticParams(E=E, nu=nu), dim=2)
    model.params = Lame(mu / 2, lam / 2)          # duck-typed D1 = lambda/2
    load = LinearLoad.assemble(m, (0.0, -3.5e7), d=2)
    v = np.ascontiguousarray(m.nodes2coord).ravel().copy()
    v[m.dofs_minim] += 1e-2 * (2.0 / nx) * (2.0 * O.uniform01(seed, m.dofs_minim) - 1.0)
    save(f"rect{nx}x{ny}_nh", **_mesh_arrays(m), **_patch_arrays(pt),
         **_evaluate(m, pt, model, load, v, 1e-8), C1=np.float64(mu / 2),
         D1=np.float64(lam / 2), nx=np.int64(nx), ny=np.int64(ny), seed=np.int64(seed))


def case_beam(nx, ny, nz, seed):
    # coordinates / connectivity from the restated generator (pinned against
    # generate_bar_mesh_3d by test_oracle_golden), everything else reference
    om = O.beam_mesh(nx, ny, nz, 0.0, 2.0, 0.0, 1.0, 0.0, 1.0)
    m = fmesh._make_mesh(3, -1, om.nodes2coord, om.elems2nodes)
    spec = fmesh.DirichletSpec([fmesh.DirichletRegion(where=lambda x: x[:, 0] < 1e-9)])
    m = fmesh.mark_dirichlet(m, spec, d=3)
    pt = femmin.build_patches(m)
    E, nu = 2e8, 0.3
    mu, lam = E / (2 * (1 + nu)), E * nu / ((1 + nu) * (1 - 2 * nu))
    model = NeoHookean(ElasticParams(E=E, nu=nu), dim=3)
    model.params = Lame(mu / 2, lam / 2)
    load = LinearLoad.assemble(m, (0.0, 0.0, -2.5e7), d=3)
    v = np.ascontiguousarray(m.nodes2coord).ravel().copy()
    v[m.dofs_minim] += 1e-2 * (2.0 / nx) * (2.0 * O.uniform01(seed, m.dofs_minim) - 1.0)
    save(f"beam{nx}x{ny}x{nz}_nh", **_mesh_arrays(m), **_patch_arrays(pt),
         **_evaluate(m, pt, model, load, v, 1e-8), C1=np.float64(mu / 2),
         D1=np.float64(lam / 2), nx=np.int64(nx), ny=np.int64(ny), nz=np.int64(nz),
         seed=np.int64(seed))


def case_lshape1_tests():
    """The reference unit-test fixture lshape_problem(1) with its rng seed."""
    m = bench.lshape_problem(1)
    pt = femmin.build_patches(m)
    rng = np.random.default_rng(20240817)
    v = rng.normal(size=m.nn)
    out = {}
    for p in (1.5, 3.0, 4.0):
        model = PLaplacian(PLaplaceParams(p=p), dim=2)
        load = LinearLoad.assemble(m, -10.0, d=1)
        r = _evaluate(m, pt, model, load, v, 1e-6)
        out.update({f"{k}_p{p:g}": val for k, val in r.items() if k != "v"})
    save("lshape1_plap", **_mesh_arrays(m), **_patch_arrays(pt), v=v, **out)


def case_small_shapes():
    """Counts and partitions of small generated meshes (mesh tests)."""
    out = {}
    for lvl in (0, 1, 2, 3):
        m = fmesh.generate_lshape_mesh_2d(lvl)
        out[f"lshape{lvl}_coords"] = m.nodes2coord
        out[f"lshape{lvl}_conn"] = m.elems2nodes
        out[f"lshape{lvl}_volumes"] = m.volumes
        out[f"lshape{lvl}_dphi"] = np.stack(m.dphi)
    save("lshape_meshes", **out)


def case_minimize():
    """The reference minimizers (solver.py) on its unit-test fixture
    lshape_problem(1): p-Laplace p = 3 (trust region and L-BFGS) and p = 2
    (against the direct Poisson solve), f = -10, v0 = 0."""
    from femmin.solver import SolveOptions, minimize
    m = bench.lshape_problem(1)
    pt = femmin.build_patches(m)
    out = {}
    for p in (3.0, 2.0):
        model = PLaplacian(PLaplaceParams(p=p), dim=2)
        load = LinearLoad.assemble(m, -10.0, d=1)

        def J(v):
            return energy(v, m, model, load)[0]

        def g(v):
            return exact_gradient(v, m, pt, model, load)

        res = minimize(J, g, np.zeros(m.nn), m.dofs_minim, SolveOptions())
        tag = f"p{p:g}"
        out.update({f"tr_u_{tag}": res.u, f"tr_J_{tag}": np.float64(res.J_u),
                    f"tr_iters_{tag}": np.int64(res.iters),
                    f"tr_ngrad_{tag}": np.int64(res.n_grad),
                    f"tr_status_{tag}": np.array(res.status)})
        if p == 3.0:
            lb = minimize(J, g, np.zeros(m.nn), m.dofs_minim,
                          SolveOptions(solver="lbfgs", tol_g=1e-8, tol_f=1e-12, tol_step=1e-8))
            out.update({"lbfgs_u_p3": lb.u, "lbfgs_J_p3": np.float64(lb.J_u)})
    out["direct_J_p2"] = np.float64(bench.poisson_solve_energy(m, f=-10.0)[1])
    out["b"] = LinearLoad.assemble(m, -10.0, d=1).b
    save("minimize_lshape1", **out)


def case_descent(nx=8, ny=4, nz=4, seed=2109, iters=20):
    """Config-5 first-order loop v <- v - alpha * grad J (masked Dirichlet
    dofs) on a small config-4/5 beam, driven by the reference's energy and
    exact_gradient; alpha = 1e-3 h / max|g0|."""
    om = O.beam_mesh(nx, ny, nz, 0.0, 2.0, 0.0, 1.0, 0.0, 1.0)
    m = fmesh._make_mesh(3, -1, om.nodes2coord, om.elems2nodes)
    spec = fmesh.DirichletSpec([fmesh.DirichletRegion(where=lambda x: x[:, 0] < 1e-9)])
    m = fmesh.mark_dirichlet(m, spec, d=3)
    pt = femmin.build_patches(m)
    E, nu = 2e8, 0.3
    mu, lam = E / (2 * (1 + nu)), E * nu / ((1 + nu) * (1 - 2 * nu))
    model = NeoHookean(ElasticParams(E=E, nu=nu), dim=3)
    model.params = Lame(mu / 2, lam / 2)
    load = LinearLoad.assemble(m, (0.0, 0.0, -2.5e7), d=3)
    v = np.ascontiguousarray(m.nodes2coord).ravel().copy()
    v[m.dofs_minim] += 1e-2 * (2.0 / nx) * (2.0 * O.uniform01(seed, m.dofs_minim) - 1.0)
    v0 = v.copy()
    alpha = 1e-3 * (2.0 / nx) / np.abs(exact_gradient(v, m, pt, model, load)).max()
    Js = []
    for _ in range(iters):
        Js.append(energy(v, m, model, load)[0])
        g = exact_gradient(v, m, pt, model, load)
        v = v.copy()
        v[m.dofs_minim] = v[m.dofs_minim] - alpha * g
    save(f"descent_beam{nx}x{ny}x{nz}", v0=v0, v_final=v, J_hist=np.array(Js),
         g_last=g, alpha=np.float64(alpha), iters=np.int64(iters), nx=np.int64(nx),
         ny=np.int64(ny), nz=np.int64(nz), seed=np.int64(seed))


def case_hessian():
    """hessian_sparsity, greedy_coloring and colored_fd_hessian (solver.py:344-398)
    of the reference on lshape_problem(1) (p = 2 at v = 0, plus the stiffness
    matrix the reference test compares with) and on the 8x4x4 config-4 beam
    (Neo-Hookean at the seeded field), gradients by the reference's
    exact_gradient."""
    from femmin.solver import colored_fd_hessian, greedy_coloring, hessian_sparsity
    out = {}
    m = bench.lshape_problem(1)
    pt = femmin.build_patches(m)
    model = PLaplacian(PLaplaceParams(p=2.0), dim=2)
    load = LinearLoad.assemble(m, -10.0, d=1)
    pat = hessian_sparsity(m, d=1)
    v = np.zeros(m.nn)

    def gx(x):
        vv = v.copy()
        vv[m.dofs_minim] = x
        return exact_gradient(vv, m, pt, model, load)

    H = colored_fd_hessian(gx, np.zeros(m.dofs_minim.size), pat, step=1e-6).toarray()
    K = bench.assemble_stiffness_matrix(m)[m.dofs_minim][:, m.dofs_minim].toarray()
    out.update(l_indptr=pat.indptr.astype(np.int64), l_indices=pat.indices.astype(np.int64),
               l_colors=greedy_coloring(pat), l_H=H, l_K=K)
    om = O.beam_mesh(8, 4, 4, 0.0, 2.0, 0.0, 1.0, 0.0, 1.0)
    bm = fmesh._make_mesh(3, -1, om.nodes2coord, om.elems2nodes)
    spec = fmesh.DirichletSpec([fmesh.DirichletRegion(where=lambda x: x[:, 0] < 1e-9)])
    bm = fmesh.mark_dirichlet(bm, spec, d=3)
    bp = femmin.build_patches(bm)
    E, nu = 2e8, 0.3
    mu, lam = E / (2 * (1 + nu)), E * nu / ((1 + nu) * (1 - 2 * nu))
    nh = NeoHookean(ElasticParams(E=E, nu=nu), dim=3)
    nh.params = Lame(mu / 2, lam / 2)
    bl = LinearLoad.assemble(bm, (0.0, 0.0, -2.5e7), d=3)
    bv = np.ascontiguousarray(bm.nodes2coord).ravel().copy()
    bv[bm.dofs_minim] += 1e-2 * (2.0 / 8) * (2.0 * O.uniform01(2109, bm.dofs_minim) - 1.0)
    bpat = hessian_sparsity(bm, d=3)

    def bgx(x):
        vv = bv.copy()
        vv[bm.dofs_minim] = x
        return exact_gradient(vv, bm, bp, nh, bl)

    bH = colored_fd_hessian(bgx, bv[bm.dofs_minim].copy(), bpat, step=1e-6).tocsr()
    bH.sort_indices()
    out.update(b_indptr=bpat.indptr.astype(np.int64), b_indices=bpat.indices.astype(np.int64),
               b_colors=greedy_coloring(bpat), b_H_indptr=bH.indptr.astype(np.int64),
               b_H_indices=bH.indices.astype(np.int64), b_H_data=bH.data, b_v=bv)
    save("hessian", **out)


def case_vtk():
    """The reference writer's bytes (vtk_io.py) for the reference test
    fixtures lshape_problem(1) (2D, point + cell data) and bar level 1 (3D)."""
    from femmin import vtk_io
    m = bench.lshape_problem(1)
    rng = np.random.default_rng(20240817)
    u = rng.normal(size=m.nn)
    dens = rng.normal(size=m.ne)
    vtk_io.write_vtk(os.path.join(HERE, "vtk_lshape1.vtk"), m.nodes2coord, m.elems2nodes,
                     point_data={"u": u}, cell_data={"density": dens})
    np.savez_compressed(os.path.join(HERE, "vtk_lshape1_data.npz"), coords=m.nodes2coord,
                        conn=m.elems2nodes, u=u, density=dens)
    b1 = bench.bar_problem(1)
    vtk_io.write_vtk(os.path.join(HERE, "vtk_bar1.vtk"), b1.nodes2coord, b1.elems2nodes)
    print("vtk fixtures written")


def case_hole(level=2, seed=2109):
    """The reference's unstructured test domain (mesh.py:246-286,
    bench.hole_problem): square with a circular hole, projected cavity nodes,
    sliver removal and node compression.  Neo-Hookean (bench's BAR_MATERIAL,
    HOLE_LOAD, Dirichlet on y = 0 and x = 0) at x + seeded noise, and a
    p-Laplace p = 3 / p = 1.8 problem on the same mesh (d = 1, same Dirichlet
    sets)."""
    m = bench.hole_problem(level)
    pt = femmin.build_patches(m)
    model = NeoHookean(bench.BAR_MATERIAL, dim=2)
    load = LinearLoad.assemble(m, bench.HOLE_LOAD, d=2)
    h = float(np.sqrt(2.0 * m.volumes.mean()))
    v = np.ascontiguousarray(m.nodes2coord).ravel().copy()
    v[m.dofs_minim] += 1e-2 * h * (2.0 * O.uniform01(seed, m.dofs_minim) - 1.0)
    out = _evaluate(m, pt, model, load, v, 1e-8)
    tol = 1e-9
    spec1 = fmesh.DirichletSpec([fmesh.DirichletRegion(where=lambda x: x[:, 1] < tol),
                                 fmesh.DirichletRegion(where=lambda x: x[:, 0] < tol)])
    m1 = fmesh.mark_dirichlet(fmesh._make_mesh(2, level, m.nodes2coord, m.elems2nodes), spec1,
                              d=1)
    p1 = femmin.build_patches(m1)
    v1 = np.zeros(m1.nn)
    v1[m1.dofs_minim] = O.uniform01(seed + 1, m1.dofs_minim)
    load1 = LinearLoad.assemble(m1, -10.0, d=1)
    extra = {}
    for p in (3.0, 1.8):
        r = _evaluate(m1, p1, PLaplacian(PLaplaceParams(p=p), dim=2), load1, v1, 1e-6)
        extra.update({f"pl{p:g}_{k}": val for k, val in r.items()})
    save(f"hole{level}", **_mesh_arrays(m), **_patch_arrays(pt), **out,
         C1=np.float64(bench.BAR_MATERIAL.C1), D1=np.float64(bench.BAR_MATERIAL.D1),
         **{"pl_" + k: val for k, val in _mesh_arrays(m1).items()},
         **{"pl_" + k: val for k, val in _patch_arrays(p1).items()}, **extra)


def case_renumbered(nx=6, ny=3, nz=3, seed=77):
    """A generic (unstructured-numbering) mesh: the config-4 beam with nodes
    and elements randomly permuted and every element's vertices rotated by an
    even permutation (orientation kept), then the reference's own
    _make_mesh (compute_p1_gradients), mark_dirichlet, build_patches and
    evaluation."""
    om = O.beam_mesh(nx, ny, nz, 0.0, 2.0, 0.0, 1.0, 0.0, 1.0)
    rng = np.random.default_rng(seed)
    nn, ne = om.nodes2coord.shape[0], om.elems2nodes.shape[0]
    pn = rng.permutation(nn)          # new node k = old node pn[k]
    inv = np.empty(nn, np.int64)
    inv[pn] = np.arange(nn)
    coords = om.nodes2coord[pn]
    conn = inv[om.elems2nodes][rng.permutation(ne)]
    rot = [(0, 1, 2, 3), (1, 2, 0, 3), (2, 0, 1, 3), (0, 2, 3, 1), (3, 1, 0, 2)]
    conn = np.stack([conn[k, list(rot[r])] for k, r in enumerate(rng.integers(0, 5, ne))])
    m = fmesh._make_mesh(3, -1, coords, conn)
    spec = fmesh.DirichletSpec([fmesh.DirichletRegion(where=lambda x: x[:, 0] < 1e-9)])
    m = fmesh.mark_dirichlet(m, spec, d=3)
    pt = femmin.build_patches(m)
    E, nu = 2e8, 0.3
    mu, lam = E / (2 * (1 + nu)), E * nu / ((1 + nu) * (1 - 2 * nu))
    model = NeoHookean(ElasticParams(E=E, nu=nu), dim=3)
    model.params = Lame(mu / 2, lam / 2)
    load = LinearLoad.assemble(m, (0.0, 0.0, -2.5e7), d=3)
    v = np.ascontiguousarray(m.nodes2coord).ravel().copy()
    v[m.dofs_minim] += 1e-2 * (2.0 / nx) * (2.0 * O.uniform01(seed, m.dofs_minim) - 1.0)
    save(f"beam{nx}x{ny}x{nz}_renumbered", **_mesh_arrays(m), **_patch_arrays(pt),
         **_evaluate(m, pt, model, load, v, 1e-8), C1=np.float64(mu / 2),
         D1=np.float64(lam / 2), perm_nodes=pn)


def case_exports(seed=5):
    """The standalone helpers of the path on reference fixtures: gather /
    evaluate_F (assembly.py:27-49), segment_sums with patch_prefix_indices
    (patches.py:74-83), linear_term (assembly.py:89-91), the nodal-f
    LinearLoad and the mass matrix (assembly.py:52-86)."""
    rng = np.random.default_rng(seed)
    out = {}
    for tag, m, d in (("l", bench.lshape_problem(2), 1), ("b", bench.bar_problem(1), 3)):
        from femmin import assembly as fas
        pt = femmin.build_patches(m)
        V = rng.normal(size=(m.nn, d))
        vals = fas.gather(V, m.elems2nodes)
        F = fas.evaluate_F(m.dphi, vals)
        rows = rng.normal(size=d * pt.total_rows)
        indx = fpatches.patch_prefix_indices(pt, d)
        f_nodal = rng.normal(size=(m.nn, d))
        load = LinearLoad.assemble(m, f_nodal, d=d)
        M = fas.assemble_mass_matrix(m)
        v = rng.normal(size=d * m.nn)
        out.update({
            f"{tag}_coords": m.nodes2coord, f"{tag}_conn": m.elems2nodes,
            f"{tag}_volumes": m.volumes, f"{tag}_dphi": np.stack(m.dphi),
            f"{tag}_V": V, f"{tag}_gather": np.stack(vals), f"{tag}_F": np.array(F),
            f"{tag}_rows": rows, f"{tag}_indx": indx,
            f"{tag}_segsum": fpatches.segment_sums(rows, indx),
            f"{tag}_f_nodal": f_nodal, f"{tag}_b_nodal": load.b,
            f"{tag}_M_indptr": M.indptr.astype(np.int64),
            f"{tag}_M_indices": M.indices.astype(np.int64), f"{tag}_M_data": M.data,
            f"{tag}_v": v, f"{tag}_linear_term": np.float64(fas.linear_term(load, v))})
    save("exports", **out)


def case_degenerate(n_cases=64, seed=3):
    """Admissibility exactly at the det F = 0 boundary (models.py:59-71,
    94-110): on the config-4 beam 4x2x2, element k's fourth node is moved onto
    the plane of its other three (v3 = v0 + s (v1 - v0) + t (v2 - v0), random
    s, t), so det F of that element is zero in exact arithmetic and a few ulps
    of either sign (or exactly 0) in numpy's six-term expansion.  Recorded per
    case: J (+inf or finite), whether exact_gradient raises, and the
    element's det as numpy computes it."""
    from femmin.models import batch_determinant
    from femmin.assembly import evaluate_F, gather, unflatten
    om = O.beam_mesh(4, 2, 2, 0.0, 2.0, 0.0, 1.0, 0.0, 1.0)
    m = fmesh._make_mesh(3, -1, om.nodes2coord, om.elems2nodes)
    spec = fmesh.DirichletSpec([fmesh.DirichletRegion(where=lambda x: x[:, 0] < 1e-9)])
    m = fmesh.mark_dirichlet(m, spec, d=3)
    pt = femmin.build_patches(m)
    E, nu = 2e8, 0.3
    mu, lam = E / (2 * (1 + nu)), E * nu / ((1 + nu) * (1 - 2 * nu))
    model = NeoHookean(ElasticParams(E=E, nu=nu), dim=3)
    model.params = Lame(mu / 2, lam / 2)
    rng = np.random.default_rng(seed)
    free = set(m.nodes_minim.tolist())
    cand = [k for k in range(m.ne) if int(m.elems2nodes[k, 3]) in free]
    vs, Js, raises, dets, elems = [], [], [], [], []
    for c in range(n_cases):
        k = cand[rng.integers(len(cand))]
        v = np.ascontiguousarray(m.nodes2coord).ravel().copy()
        n0, n1, n2, n3 = (int(x) for x in m.elems2nodes[k])
        s, t = rng.uniform(0.1, 0.6, 2)
        V = v.reshape(-1, 3)
        V[n3] = V[n0] + s * (V[n1] - V[n0]) + t * (V[n2] - V[n0])
        if c % 4 == 3:  # a hair off the plane: det ~ +-1e-16
            V[n3] += rng.choice([-1.0, 1.0]) * 1e-16 * rng.uniform(0, 4, 3)
        J, W = energy(v, m, model)
        try:
            exact_gradient(v, m, pt, model)
            r = False
        except InadmissibleStateError:
            r = True
        F = evaluate_F(m.dphi, gather(unflatten(v, 3), m.elems2nodes))
        det = batch_determinant(F)
        vs.append(v)
        Js.append(J)
        raises.append(r)
        dets.append(det[k])
        elems.append(k)
    save("degenerate_beam4x2x2", **_mesh_arrays(m), **_patch_arrays(pt), v=np.array(vs),
         J=np.array(Js), raises=np.array(raises), det=np.array(dets), elem=np.array(elems),
         C1=np.float64(mu / 2), D1=np.float64(lam / 2))


if __name__ == "__main__":
    if len(sys.argv) > 1:  # only the named cases, e.g. "descent"
        for name in sys.argv[1:]:
            globals()["case_" + name]()
        sys.exit(0)
    case_hole()
    case_renumbered()
    case_exports()
    case_degenerate()
    case_hessian()
    case_vtk()
    case_descent()
    case_minimize()
    case_small_shapes()
    case_lshape1_tests()
    case_lshape(4, 3.0, 2109, "cfg1_lshape4_p3")
    case_lshape(4, 1.8, 2110, "lshape4_p1.8")
    case_bar_twist()
    case_bar2_mesh()
    case_rect(32, 16, 2109)
    case_beam(8, 4, 4, 2109)
