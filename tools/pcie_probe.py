"""Pinned-host copy rates on this box: H2D alone, D2H alone, both at once."""
import torch

n = 100 * 1024 * 1024 // 8
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_in = torch.empty(n, dtype=torch.float64, device="cuda")
d_out = torch.zeros(n, dtype=torch.float64, device="cuda")
up, down = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    up.wait_stream(torch.cuda.current_stream())
    down.wait_stream(torch.cuda.current_stream())
    for _ in range(reps):
        fn()
    torch.cuda.current_stream().wait_stream(up)
    torch.cuda.current_stream().wait_stream(down)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def h2d():
    with torch.cuda.stream(up):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(down):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d()
    d2h()


B = n * 8
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    ms = timed(fn)
    print(f"{name}: {ms:.3f} ms per 100 MiB -> {B / ms / 1e6:.1f} GB/s per direction")
