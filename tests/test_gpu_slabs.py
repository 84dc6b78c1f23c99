"""SURVEY §8e parity on the GPU: x1-slab ranks evaluated by the CUDA kernels
(problems.beam(ix0, ix1) + DeviceMesh) and reduced by parallel.SlabExchange
must reproduce the single-domain J and exact gradient, and the config-5
descent loop with the exchange must track the single-domain loop.  One GPU:
the ranks share it over gloo (host-staged exchange), which checks the
algebra and the exchange wiring, not NCCL performance."""

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


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, outdir, alpha):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2109_01158_b200 import problems
    from paper_2109_01158_b200.parallel import SlabExchange, slab_range
    ix0, ix1 = slab_range(NX, rank, world)
    pr = problems.beam(NX, NY, NZ, seed=5, ix0=ix0, ix1=ix1)
    ex = SlabExchange.from_problem(pr, rank, world)
    J = torch.empty(3, dtype=torch.float64, device="cuda")
    g = pr.dm.exact_gradient(pr.v, pr.model, pr.b, J=J)
    ex.reduce(g, J)
    v = pr.v.clone()
    Jh = torch.empty((ITERS, 3), dtype=torch.float64, device="cuda")
    pr.dm.descent(v, pr.model, pr.b, alpha, ITERS, J_hist=Jh, exchange=ex)
    pr.dm.check()
    nxl = ix1 - ix0
    dm_ = pr.meta["dofs_minim"].cpu().numpy()
    local = dm_ // 3
    gid = (local % (nxl + 1) + ix0) + (NX + 1) * (local // (nxl + 1))
    np.savez(os.path.join(outdir, f"r{rank}.npz"), g=g.cpu().numpy(), J=J.cpu().numpy(),
             gdof=3 * gid + dm_ % 3, Jh=Jh.cpu().numpy(), v=v.cpu().numpy(),
             vdof=(lambda n: 3 * ((n % (nxl + 1) + ix0) + (NX + 1) * (n // (nxl + 1))))(
                 np.arange(v.numel()) // 3) + np.arange(v.numel()) % 3)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gpu_slabs_reproduce_single_domain(tmp_path, world):
    from paper_2109_01158_b200 import problems
    pr = problems.beam(NX, NY, NZ, seed=5, keep=True)
    J = torch.empty(3, dtype=torch.float64, device="cuda")
    gg = pr.dm.exact_gradient(pr.v, pr.model, pr.b, J=J).cpu().numpy()
    Jg = J.cpu().numpy()
    alpha = 1e-3 * (2.0 / NX) / float(np.abs(gg).max())
    v = pr.v.clone()
    Jh = torch.empty((ITERS, 3), dtype=torch.float64, device="cuda")
    pr.dm.descent(v, pr.model, pr.b, alpha, ITERS, J_hist=Jh)
    Jh, vg = Jh.cpu().numpy(), v.cpu().numpy()
    pos = {int(d): k for k, d in enumerate(pr.meta["dofs_minim"].cpu().numpy())}
    del pr
    torch.cuda.synchronize()
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), alpha), nprocs=world, join=True)
    scale = np.abs(gg).max()
    for r in range(world):
        z = np.load(tmp_path / f"r{r}.npz")
        idx = np.array([pos[int(x)] for x in z["gdof"]])
        assert np.abs(z["g"] - gg[idx]).max() / scale < 1e-13
        assert abs(z["J"][0] - Jg[0]) / abs(Jg[0]) < 1e-13
        np.testing.assert_allclose(z["Jh"][:, 0], Jh[:, 0], rtol=1e-13)
        assert np.abs(z["v"] - vg[z["vdof"]]).max() <= 1e-13 * np.abs(vg).max()
    # every rank holds the same J bits (rank-order sum of the gathered partials)
    J0 = np.load(tmp_path / "r0.npz")["J"]
    for r in range(1, world):
        np.testing.assert_array_equal(np.load(tmp_path / f"r{r}.npz")["J"], J0)
