"""The C-ABI slab exchange (fm_slab_*, csrc/fm_slab.cu) on a real GPU with a
one-rank NCCL communicator: run-time NCCL resolution, communicator set-up, the
grouped launch and the fixed-order J sum (a single rank has no planes, so g
is untouched and J = its own partial).  The two-neighbour plane exchange needs
two GPUs; its host logic is covered by tests/test_slab_gloo.py."""

import os
import socket

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_native_slab_single_rank():
    from paper_2109_01158_b200 import problems
    from paper_2109_01158_b200.parallel import SlabExchange
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        pr = problems.beam(8, 4, 4, seed=3, ix0=0, ix1=8)
        ex = SlabExchange.from_problem(pr, 0, 1)
        assert ex.native is not None
        J = torch.empty(3, dtype=torch.float64, device="cuda")
        g = pr.dm.exact_gradient(pr.v, pr.model, pr.b, J=J)
        g0, J0 = g.clone(), J.clone()
        for _ in range(3):  # repeated launches reuse the communicator
            ex.reduce(g, J)
        torch.cuda.synchronize()
        assert torch.equal(g, g0) and torch.equal(J, J0)
        ex.reduce(None, J)
        torch.cuda.synchronize()
        assert torch.equal(J, J0)
    finally:
        dist.destroy_process_group()


def test_step_graph_capture():
    """The fused evaluation and the C-ABI exchange are capture-safe: one CUDA
    graph of (tile kernel, finishing pass, pack, grouped NCCL, unpack) replays
    to the eager results bit for bit (what bench.py uses for N > 1 ranks)."""
    from paper_2109_01158_b200 import problems
    from paper_2109_01158_b200.parallel import SlabExchange
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        pr = problems.beam(12, 6, 6, seed=4)
        ex = SlabExchange.from_problem(pr, 0, 1)
        g = torch.empty(pr.dm.nfree_dofs, dtype=torch.float64, device="cuda")
        J = torch.empty(3, dtype=torch.float64, device="cuda")

        def step():
            pr.dm.exact_gradient(pr.v, pr.model, pr.b, g=g, J=J)
            ex.reduce(g, J)

        step()
        torch.cuda.synchronize()
        g_ref, J_ref = g.clone(), J.clone()
        graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            step()  # warm-up on the capture stream
        torch.cuda.current_stream().wait_stream(side)
        with torch.cuda.graph(graph):
            step()
        for _ in range(3):
            g.zero_()
            J.zero_()
            graph.replay()
            torch.cuda.synchronize()
            assert torch.equal(g, g_ref) and torch.equal(J, J_ref)
        pr.dm.check()
    finally:
        dist.destroy_process_group()
