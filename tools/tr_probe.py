"""Where does the device minimizer's time go (config 4)?"""
import sys, time, torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2109_01158_b200 import problems
from paper_2109_01158_b200.solver import SolveOptions, minimize_device
pr = problems.beam(256, 128, 128, seed=2109)
dm, model, b, v = pr.dm, pr.model, pr.b, pr.v
dofs = pr.meta["dofs_minim"]
for rep in range(2):
    res = minimize_device(dm, model, b, v, dofs, SolveOptions(max_iters=3, max_cg=20))
    print("run", rep, "time", res.time, "grad calls", res.n_grad, "energy calls", res.n_energy)
x = v.index_select(0, dofs)
work = v.clone()
def t(fn, n=10):
    fn(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / n * 1e3
print("grad only (kernels)", t(lambda: dm.exact_gradient(v, model, b)))
print("grad + check", t(lambda: (dm.exact_gradient(v, model, b), dm.check())))
print("embed", t(lambda: work.index_copy_(0, dofs, x)))
print("energy + item", t(lambda: float(dm.energy(v, model, b)[0])))
print("dot item", t(lambda: float(torch.dot(x, x))))
print("norm item", t(lambda: float(torch.linalg.vector_norm(x))))
print("axpy", t(lambda: x + 1e-3 * x))
