"""Full-size parity of the GPU preprocessing (BASELINE configs 2-4 at their
real sizes): every index structure the GPU builds — coordinates,
connectivity, Dirichlet partitions, the patch CSR (prefix / elems / slot) and
the seeded trial field — bit for bit against the CPU oracle's restatement of
mesh.py:177-221 / 125-174 / 289-322 and patches.py:37-71 (the oracle is
pinned to the reference by tests/test_oracle_golden.py), plus P1 data and
the load vector to rounding.  Separately (``test_gpu_parity``), the
evaluation at these sizes is checked at sampled dofs.

These build the full meshes on the host too (cfg4: ~10 GB, ~40 s).
"""

import numpy as np
import pytest

from oracle import femmin_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2109_01158_b200 import problems  # noqa: E402


def _host(t):
    return t.cpu().numpy()


def _compare(pr, om, v_ref, f):
    mt = pr.meta
    np.testing.assert_array_equal(_host(mt["coords"]), om.nodes2coord)
    np.testing.assert_array_equal(_host(mt["conn"]), om.elems2nodes)
    for k in ("nodes_minim", "dofs_minim", "dofs_minim_local", "dofs_dirichlet"):
        np.testing.assert_array_equal(_host(mt[k]), getattr(om, k), err_msg=k)
    np.testing.assert_array_equal(_host(mt["nodes_dirichlet_idx"]), om.nodes_dirichlet)
    P = O.build_patches(om)
    np.testing.assert_array_equal(_host(mt["p_prefix"]), P.prefix)
    np.testing.assert_array_equal(_host(mt["p_elems"]), P.elems)
    np.testing.assert_array_equal(_host(mt["p_slot"]), P.slot)
    np.testing.assert_array_equal(_host(pr.v), v_ref)
    # P1 data: closed form vs LAPACK (ulps)
    vol = _host(mt["volumes"])
    np.testing.assert_allclose(vol, om.volumes, rtol=1e-12)
    dphi = _host(mt["dphi"])
    ref = np.stack(om.dphi)
    assert np.abs(dphi - ref).max() <= 1e-12 * np.abs(ref).max()
    # constant-f load: b_i = f_j * sum_{k ∋ i} |T_k| / (dim+1) (assembly.py:65-82)
    nv = om.elems2nodes.shape[1]
    w = np.bincount(om.elems2nodes.ravel(), weights=np.repeat(om.volumes / nv, nv),
                    minlength=om.nodes2coord.shape[0])
    b_ref = (w[:, None] * np.asarray(f)[None, :]).ravel()
    b = _host(pr.b)
    assert np.abs(b - b_ref).max() <= 1e-13 * np.abs(b_ref).max()


def test_cfg3_full_structures_bit_exact():
    """Config 3 (2048 x 1024 rectangle, 4.2 M triangles)."""
    pr = problems.CONFIGS["cfg3"](keep=True)
    om, _, _, v = O.problem_rect(2048, 1024, seed=2109)
    _compare(pr, om, v, [0.0, -3.5e7])


def test_cfg2_full_structures_bit_exact():
    """Config 2 (L-shape level 10, 25.2 M triangles): mesh.py:200-221 with
    np.unique node compression, full-boundary Dirichlet."""
    pr = problems.CONFIGS["cfg2"](keep=True)
    om = O.lshape_mesh(10)
    om = O.mark_dirichlet(om, O.fixed_mask(om, [(O.lshape_boundary(10), None)], 1), 1)
    _compare(pr, om, O.field_plap(om, 2109), [-10.0])


def test_cfg4_full_structures_bit_exact():
    """Config 4 (256 x 128 x 128 Kuhn beam, 25.2 M tetrahedra)."""
    pr = problems.CONFIGS["cfg4"](keep=True)
    om = O.beam_mesh(256, 128, 128, 0.0, 2.0, 0.0, 1.0, 0.0, 1.0)
    om = O.mark_dirichlet(om, O.fixed_mask(om, [(O.left_face, None)], 3), 3)
    v = np.ascontiguousarray(om.nodes2coord).ravel().copy()
    dof = om.dofs_minim
    v[dof] = v[dof] + 1e-2 * (2.0 / 256) * (2.0 * O.uniform01(2109, dof) - 1.0)
    _compare(pr, om, v, [0.0, 0.0, -2.5e7])
