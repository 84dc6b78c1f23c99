"""Multi-rank x1-slab partition on CPU (gloo, world size 2 and 3): the host-side
exchange of paper_2109_01158_b200.parallel with slab-local partials from the
oracle must reproduce the single-domain J and exact gradient."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import femmin_oracle as O

NX, NY, NZ = 12, 4, 4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2109_01158_b200.parallel import SlabExchange, slab_range
    ix0, ix1 = slab_range(NX, rank, world)
    m, model, b, v = O.problem_beam(NX, NY, NZ, seed=11, ix0=ix0, ix1=ix1)
    P = O.build_patches(m)
    J, W = O.energy(v, m, model, b)
    A = float(m.volumes @ W)
    C = float(b @ v)
    g = torch.from_numpy(O.exact_gradient(v, m, P, model, b).copy())
    Jt = torch.tensor([J, A, C], dtype=torch.float64)
    ex = SlabExchange(NX, NY, NZ, ix0, ix1, 3, torch.from_numpy(m.dofs_minim), rank, world)
    ex.reduce(g, Jt)
    nxl = ix1 - ix0
    local = np.arange(m.nn)
    gid = (local % (nxl + 1) + ix0) + (NX + 1) * (local // (nxl + 1))
    gdof = 3 * gid[m.dofs_minim // 3] + m.dofs_minim % 3
    np.savez(os.path.join(outdir, f"r{rank}.npz"), g=g.numpy(), J=Jt.numpy(), gdof=gdof)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_exchange_reproduces_global(tmp_path, world):
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    m, model, b, v = O.problem_beam(NX, NY, NZ, seed=11)
    P = O.build_patches(m)
    Jg = O.energy(v, m, model, b)[0]
    gg = O.exact_gradient(v, m, P, model, b)
    pos = {int(dof): k for k, dof in enumerate(m.dofs_minim)}
    scale = np.abs(gg).max()
    Js = []
    for r in range(world):
        z = np.load(tmp_path / f"r{r}.npz")
        Js.append(z["J"])
        idx = np.array([pos[int(x)] for x in z["gdof"]])
        assert np.abs(z["g"] - gg[idx]).max() / scale < 1e-12
    # identical J on every rank (rank-order sum), equal to the global J
    for r in range(1, world):
        np.testing.assert_array_equal(Js[r], Js[0])
    assert abs(Js[0][0] - Jg) / abs(Jg) < 1e-12


def test_slab_ranges_cover_and_balance():
    from paper_2109_01158_b200.parallel import slab_range
    for nx, world in ((256, 8), (1024, 8), (256, 3)):
        rs = [slab_range(nx, r, world) for r in range(world)]
        assert rs[0][0] == 0 and rs[-1][1] == nx
        assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
        sizes = [b - a for a, b in rs]
        assert max(sizes) - min(sizes) <= 1


def test_slab_oracle_mesh_is_a_restriction():
    """The slab generator reproduces the global mesh's coordinates and
    connectivity (renumbered), so slab partials are exact partial sums."""
    m = O.beam_mesh(NX, NY, NZ, 0.0, 2.0, 0.0, 1.0, 0.0, 1.0)
    s = O.beam_mesh(NX, NY, NZ, 0.0, 2.0, 0.0, 1.0, 0.0, 1.0, ix0=4, ix1=9)
    nxl = 5
    local = np.arange(s.nn)
    gid = (local % (nxl + 1) + 4) + (NX + 1) * (local // (nxl + 1))
    np.testing.assert_array_equal(s.nodes2coord, m.nodes2coord[gid])
    cubes = np.array([cx + NX * (cy + NY * cz) for cz in range(NZ) for cy in range(NY)
                      for cx in range(4, 9)])
    gel = (6 * cubes[:, None] + np.arange(6)[None]).ravel()
    np.testing.assert_array_equal(gid[s.elems2nodes], m.elems2nodes[gel])


def test_stack_ranges_cover_and_fill_boxes():
    """Sub-slab cuts (parallel.stack_ranges): contiguous, covering, near
    equal; large sub-slabs fill whole 8-layer tile boxes except the last."""
    from paper_2109_01158_b200.parallel import stack_ranges
    for ix0, ix1, k in [(0, 512, 6), (512, 1024, 6), (0, 512, 17), (256, 512, 4),
                        (0, 24, 3), (12, 24, 2), (0, 24, 5), (0, 8, 3), (3, 4, 1)]:
        r = stack_ranges(ix0, ix1, k)
        assert len(r) == min(k, ix1 - ix0) and r[0][0] == ix0 and r[-1][1] == ix1
        assert all(a < z for a, z in r) and all(r[i][1] == r[i + 1][0] for i in range(len(r) - 1))
        n = [z - a for a, z in r]
        assert max(n) - min(n) <= max(12, (ix1 - ix0) // k // 4)
        if ix1 - ix0 >= 16 * k:
            for a, z in r[:-1]:
                assert ((z - a) + (0 if a == 0 else 1)) % 8 == 0
