import time, torch, numpy as np
from concurrent.futures import ThreadPoolExecutor
n = 12_830_211
a = np.random.rand(n)
d = torch.empty(n, dtype=torch.float64, device="cuda")
def t(f, k=10):
    f(); torch.cuda.synchronize()
    t0=time.perf_counter()
    for _ in range(k): f()
    torch.cuda.synchronize(); return (time.perf_counter()-t0)/k*1e3
print("pageable H2D from numpy", t(lambda: d.copy_(torch.from_numpy(a))))
print("pageable D2H new array", t(lambda: d.cpu().numpy()))
pin = torch.empty(n, dtype=torch.float64, pin_memory=True)
print("np.copyto into pinned", t(lambda: np.copyto(pin.numpy(), a)))
ex = ThreadPoolExecutor(8)
def pcopy(dst, src, parts=8):
    k = len(src); cuts=[k*i//parts for i in range(parts+1)]
    list(ex.map(lambda i: np.copyto(dst[cuts[i]:cuts[i+1]], src[cuts[i]:cuts[i+1]]), range(parts)))
print("parallel copyto into pinned", t(lambda: pcopy(pin.numpy(), a)))
print("pinned H2D", t(lambda: d.copy_(pin, non_blocking=True)))
def d2h_pinned():
    o = torch.empty(n, dtype=torch.float64, pin_memory=True); o.copy_(d, non_blocking=True); torch.cuda.current_stream().synchronize(); return o.numpy()
print("D2H into fresh pinned (caching allocator)", t(d2h_pinned))
print("nproc", __import__('os').cpu_count())
