import sys, time, torch
sys.path.insert(0, '/root/repo')
from paper_2109_01158_b200 import problems
from paper_2109_01158_b200.solver import _DeviceSteihaug, SolveOptions
pr = problems.CONFIGS["cfg4"](keep=True)
dm, model, b, v = pr.dm, pr.model, pr.b, pr.v
dofs = pr.meta["dofs_minim"]
work = v.clone()
count = {"g": 0}
def embed(x):
    return work.index_copy_(0, dofs, x)
cg = _DeviceSteihaug(dm, model, b, work, count, False, embed)
x = v.index_select(0, dofs)
g = dm.exact_gradient(v, model, b)
torch.cuda.synchronize()
for it in (2, 5, 10, 20):
    count["g"] = 0
    torch.cuda.synchronize(); t0 = time.perf_counter()
    p, hit = cg.solve(g, x, float(torch.linalg.vector_norm(x)), 1e10, 1e-30, it)
    torch.cuda.synchronize(); t = time.perf_counter() - t0
    print(f"maxiter {it}: {t*1e3:.2f} ms, {count['g']} grads, {t*1e3/max(1,count['g']):.3f} ms/grad")
# pieces
import ctypes
torch.cuda.synchronize(); t0=time.perf_counter()
for _ in range(20): dm.exact_gradient(work, model, b, g=cg.gp)
torch.cuda.synchronize(); print("grad only", (time.perf_counter()-t0)/20*1e3)
lib = cg.lib; P = cg._p
from paper_2109_01158_b200._device import stream_ptr
torch.cuda.synchronize(); t0=time.perf_counter()
for _ in range(20): lib.fm_cg_embed(dm._h, P(x), P(cg.d), P(cg.st), 1, 1.0, P(work), stream_ptr())
torch.cuda.synchronize(); print("embed", (time.perf_counter()-t0)/20*1e3)
cg.st[16] = 0
torch.cuda.synchronize(); t0=time.perf_counter()
for _ in range(20): lib.fm_cg_iterate(cg.n, P(cg.gp), P(cg.gm), P(cg.Hd), P(cg.z), P(cg.znew), P(cg.r), P(cg.d), P(cg.st), P(cg.part), P(cg.ticket), stream_ptr())
torch.cuda.synchronize(); print("iterate (3 kernels)", (time.perf_counter()-t0)/20*1e3)
torch.cuda.synchronize(); t0=time.perf_counter()
for _ in range(20): cg._done()
print("done check", (time.perf_counter()-t0)/20*1e3)
