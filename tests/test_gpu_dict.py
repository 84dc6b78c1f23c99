"""Record dictionaries of the fused tile kernel (csrc/fm_ctx.cuh DICT_MAX):
tiles whose own elements share at most 16 distinct (vol, dphi) records stream
one slot byte per element and read the record from a per-tile table.  The
records are the same bits either way, so every evaluation (gradients.py:124-149
exact, 84-121 FD, assembly.py:94-106 energy, the Hessian-vector product) must be
bitwise equal with the dictionaries on (default) and off (FM_TILE_DICT=0).
Grids with a power-of-two spacing (every benchmark config) have bit-identical
records from cube to cube and must be coded; the reference's unstructured hole
mesh must fall back to streamed records for its tiles with more distinct
records (as do grids whose spacing rounds differently from cell to cell)."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2109_01158_b200 as fb  # noqa: E402
from paper_2109_01158_b200 import problems  # noqa: E402


def _build(make, dict_on):
    old = os.environ.get("FM_TILE_DICT")
    os.environ["FM_TILE_DICT"] = "1" if dict_on else "0"
    try:
        return make()
    finally:
        if old is None:
            del os.environ["FM_TILE_DICT"]
        else:
            os.environ["FM_TILE_DICT"] = old


def _all_outputs(pr, eps):
    dm = pr.dm
    J = torch.empty(3, dtype=torch.float64, device="cuda")
    g = dm.exact_gradient(pr.v, pr.model, pr.b, J=J).clone()
    g0 = dm.exact_gradient(pr.v, pr.model, pr.b).clone()
    Je = torch.empty(3, dtype=torch.float64, device="cuda")
    dens = torch.empty(dm.ne, dtype=torch.float64, device="cuda")
    dm.energy(pr.v, pr.model, pr.b, densities=dens, out=Je)
    gfd = dm.numeric_gradient(pr.v, pr.model, pr.b, eps).clone()
    # a direction on the free dofs, zero on the Dirichlet dofs
    gen = torch.Generator(device="cuda").manual_seed(5)
    xp = torch.rand(dm.nfree_dofs, generator=gen, device="cuda", dtype=torch.float64) - 0.5
    p = torch.zeros(pr.v.numel(), dtype=torch.float64, device="cuda")
    p[pr.meta["dofs_minim"]] = xp
    hp = dm.hvp(pr.v, p, pr.model).clone()
    dm.check()
    torch.cuda.synchronize()
    return [x.cpu().numpy() for x in (J, g, g0, Je, dens, gfd, hp)]


@pytest.mark.parametrize("name,make,eps", [
    ("beam", lambda: problems.beam(64, 32, 32, seed=7, keep=True), 1e-8),
    ("lshape", lambda: problems.lshape(7, 3.0, seed=7, keep=True), 1e-6),
    ("rect", lambda: problems.rect(256, 128, seed=7, keep=True), 1e-8),
])
def test_dictionary_coded_tiles_give_the_same_bits(name, make, eps):
    on = _build(make, True)
    off = _build(make, False)
    assert on.dm.stats["dict_tiles"] > 0, "a power-of-two grid must be dictionary-coded"
    # (tiles whose elements all belong to other tiles have nothing to code)
    assert on.dm.stats["dict_tiles"] >= 0.5 * on.dm.stats["n_tiles"]
    assert off.dm.stats["dict_tiles"] == 0
    a, b = _all_outputs(on, eps), _all_outputs(off, eps)
    for what, x, y in zip(("J", "g (with J)", "g", "J energy", "densities", "FD g", "Hp"), a, b):
        assert np.array_equal(x, y), f"{name}: {what} differs between coded and streamed records"


def test_mixed_context_gives_the_same_bits():
    """A beam whose spacing (1/24) rounds differently from cell to cell: only a
    few tiles have <= 16 distinct records, so coded and streamed tiles share
    one launch (and the stages keep their full record area)."""
    make = lambda: problems.beam(48, 24, 24, seed=11, keep=True)  # noqa: E731
    on = _build(make, True)
    off = _build(make, False)
    assert 0 < on.dm.stats["dict_tiles"] < on.dm.stats["n_tiles"]
    a, b = _all_outputs(on, 1e-8), _all_outputs(off, 1e-8)
    for what, x, y in zip(("J", "g (with J)", "g", "J energy", "densities", "FD g", "Hp"), a, b):
        assert np.array_equal(x, y), f"{what} differs between coded and streamed records"


def test_unstructured_mesh_falls_back(golden):
    """The hole mesh (mesh.py:246-286): its triangles are all different, so no
    tile beyond the tiny ones can be coded; the evaluation itself is checked
    against the reference in test_gpu_generic.py (default build = dictionaries on)."""
    from paper_2109_01158_b200 import device as fdev
    g = golden("hole2")
    m = fb.Mesh(dim=2, level=-1, nodes2coord=g["coords"], elems2nodes=g["conn"],
                volumes=g["volumes"], dphi=list(g["dphi"]), d=int(g["d"]),
                nodes_dirichlet=g["nodes_dirichlet"], nodes_minim=g["nodes_minim"],
                dofs_dirichlet=g["dofs_dirichlet"], dofs_minim=g["dofs_minim"],
                dofs_minim_local=g["dofs_minim_local"])
    dm = fdev.context_for(m, None, 2)
    assert dm.stats["dict_tiles"] < dm.stats["n_tiles"]
