"""Sub-slab stacks (parallel.SlabStack): a slab held as K evaluation contexts
on one GPU must reproduce the single-domain J, exact and FD gradients, the
energy and the config-5 descent loop; the interface copies shared by two
sub-slabs must stay bitwise equal.  Also a 2-rank gloo split whose ranks are
stacks (the config-5 2-GPU layout in miniature)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

NX, NY, NZ = 24, 8, 8
ITERS = 5


def _global_dofs(nx, ny, ix0, ix1, dofs_minim):
    """slab-local free dofs -> global dofs of the (nx, ny, nz) beam"""
    nxl = ix1 - ix0
    local = dofs_minim // 3
    gid = (local % (nxl + 1) + ix0) + (nx + 1) * (local // (nxl + 1))
    return 3 * gid + dofs_minim % 3


def _stack_gdofs(st):
    """global dof of every position of the stack's concatenated gradient"""
    out = []
    for (a, z), m in zip(st.ranges, st.dms):
        dm_ = m.nodes_minim  # free nodes; all 3 components free off x1 = 0
        nodes = dm_.cpu().numpy()
        dofs = (3 * nodes[:, None] + np.arange(3)[None]).reshape(-1)
        out.append(_global_dofs(st.nx, st.ny, a, z, dofs))
    return np.concatenate(out)


def _single(seed=5):
    from paper_2109_01158_b200 import problems
    pr = problems.beam(NX, NY, NZ, seed=seed, keep=True)
    J = torch.empty(3, dtype=torch.float64, device="cuda")
    g = pr.dm.exact_gradient(pr.v, pr.model, pr.b, J=J).cpu().numpy()
    gfd = pr.dm.numeric_gradient(pr.v, pr.model, pr.b, 1e-8).cpu().numpy()
    E = pr.dm.energy(pr.v, pr.model, pr.b).cpu().numpy().copy()
    pos = {int(d): k for k, d in enumerate(pr.meta["dofs_minim"].cpu().numpy())}
    return pr, J.cpu().numpy(), g, gfd, E, pos


@pytest.mark.parametrize("parts", [2, 3, 5])
def test_stack_reproduces_single_domain(parts):
    from paper_2109_01158_b200.parallel import SlabStack
    pr, Jg, gg, gfd, Eg, pos = _single()
    st = SlabStack(NX, NY, NZ, 0, NX, parts, seed=5)
    assert st.K == parts and st.ne == pr.ne
    J = torch.empty(3, dtype=torch.float64, device="cuda")
    g = st.exact_gradient(st.V, st.model, st.B, J=J).cpu().numpy()
    st.check()
    gd = _stack_gdofs(st)
    idx = np.array([pos[int(x)] for x in gd])
    scale = np.abs(gg).max()
    assert np.abs(g - gg[idx]).max() / scale < 1e-13
    assert abs(J.cpu().numpy()[0] - Jg[0]) / abs(Jg[0]) < 1e-13
    # both copies of every interface dof hold the same bits
    gt = torch.from_numpy(g)
    assert torch.equal(gt[st.pa.cpu()], gt[st.pb.cpu()])
    # gradient without J, energy, FD
    g2 = st.exact_gradient(st.V, st.model, st.B).cpu().numpy()
    np.testing.assert_array_equal(g2, g)
    E = st.energy(st.V, st.model, st.B).cpu().numpy()
    assert abs(E[0] - Eg[0]) / abs(Eg[0]) < 1e-13
    f = st.numeric_gradient(st.V, st.model, st.B, 1e-8).cpu().numpy()
    fs = np.abs(gfd).max()
    assert np.abs(f - gfd[idx]).max() / fs < 1e-9  # FD roundoff of the two sums
    st.check()
    # kernel timing hooks
    a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.time_next(a, z)
    st.exact_gradient(st.V, st.model, st.B, J=J)
    km = st.kernel_ms()
    assert len(km) == 1 and km[0] > 0


def test_stack_descent_matches_single_domain():
    from paper_2109_01158_b200.parallel import SlabStack
    pr, Jg, gg, _, _, pos = _single()
    alpha = 1e-3 * (2.0 / NX) / float(np.abs(gg).max())
    v = pr.v.clone()
    Jh = torch.empty((ITERS, 3), dtype=torch.float64, device="cuda")
    pr.dm.descent(v, pr.model, pr.b, alpha, ITERS, J_hist=Jh)
    st = SlabStack(NX, NY, NZ, 0, NX, 3, seed=5)
    vs = st.V.clone()
    Jhs = torch.empty((ITERS, 3), dtype=torch.float64, device="cuda")
    st.descent(vs, st.model, st.B, alpha, ITERS, J_hist=Jhs)
    st.check()
    np.testing.assert_allclose(Jhs[:, 0].cpu().numpy(), Jh[:, 0].cpu().numpy(), rtol=1e-13)
    # the stack's field blocks against the single-domain field
    vg = v.cpu().numpy()
    for k, (a, z) in enumerate(st.ranges):
        vk = vs[st.voff[k]:st.voff[k + 1]].cpu().numpy()
        n = np.arange(vk.size) // 3
        nxl = z - a
        gid = (n % (nxl + 1) + a) + (NX + 1) * (n // (nxl + 1))
        assert np.abs(vk - vg[3 * gid + np.arange(vk.size) % 3]).max() <= 1e-13 * np.abs(vg).max()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from types import SimpleNamespace

    from paper_2109_01158_b200.parallel import SlabExchange, SlabStack, slab_range
    ix0, ix1 = slab_range(NX, rank, world)
    st = SlabStack(NX, NY, NZ, ix0, ix1, 2, seed=5)
    ex = SlabExchange.from_problem(SimpleNamespace(dm=st), rank, world)
    J = torch.empty(3, dtype=torch.float64, device="cuda")
    g = st.exact_gradient(st.V, st.model, st.B, J=J)
    ex.reduce(g, J)
    st.check()
    np.savez(os.path.join(outdir, f"r{rank}.npz"), g=g.cpu().numpy(), J=J.cpu().numpy(),
             gdof=_stack_gdofs(st))
    dist.destroy_process_group()


def test_ranks_of_stacks_reproduce_single_domain(tmp_path):
    pr, Jg, gg, _, _, pos = _single()
    del pr
    torch.cuda.synchronize()
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    scale = np.abs(gg).max()
    for r in range(world):
        z = np.load(tmp_path / f"r{r}.npz")
        idx = np.array([pos[int(x)] for x in z["gdof"]])
        assert np.abs(z["g"] - gg[idx]).max() / scale < 1e-13
        assert abs(z["J"][0] - Jg[0]) / abs(Jg[0]) < 1e-13


def test_stack_mid_size_matches_single_domain():
    """A 96x48x48 beam (1.3 M tets, many tiles per sub-slab) as 4 sub-slabs."""
    from paper_2109_01158_b200 import problems
    from paper_2109_01158_b200.parallel import SlabStack
    nx, ny, nz = 96, 48, 48
    pr = problems.beam(nx, ny, nz, seed=7, keep=True)
    J = torch.empty(3, dtype=torch.float64, device="cuda")
    gg = pr.dm.exact_gradient(pr.v, pr.model, pr.b, J=J).cpu().numpy()
    Jg = J.cpu().numpy().copy()
    pos = {int(d): k for k, d in enumerate(pr.meta["dofs_minim"].cpu().numpy())}
    del pr
    st = SlabStack(nx, ny, nz, 0, nx, 4, seed=7)
    g = st.exact_gradient(st.V, st.model, st.B, J=J).cpu().numpy()
    st.check()
    idx = np.array([pos[int(x)] for x in _stack_gdofs(st)])
    assert np.abs(g - gg[idx]).max() / np.abs(gg).max() < 1e-13
    assert abs(J.cpu().numpy()[0] - Jg[0]) / abs(Jg[0]) < 1e-13
