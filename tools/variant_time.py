"""A/B timing of library variants (profiling aid).

    python tools/variant_time.py --config cfg4 lib=product lib=fdiff:FM_OWNER_RULE=0 ...

Each argument is ``lib=<variant>[:ENV=VAL;...]``: ``product`` is
lib/libfemmin_b200.so, any other name lib/libfemmin_<name>.so (built here
beforehand with paper_2109_01158_b200.build.build_variant).  Every variant runs
in its own process: the fused J + exact gradient is timed (CUDA events, 50
evaluations after warm-up, whole evaluation and the tile kernel alone) and
compared with the first variant's gradient.  ``--op fd`` times the FD
gradient instead (eps 1e-8, 1e-6 for scalar fields)."""
import argparse
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json, torch
sys.path.insert(0, %r)
from paper_2109_01158_b200 import problems
pr = problems.CONFIGS[%r]()
g = torch.empty(pr.dm.nfree_dofs, dtype=torch.float64, device="cuda")
J = torch.empty(3, dtype=torch.float64, device="cuda")
OP = %r
EPS = 1e-6 if pr.dm.d == 1 else 1e-8
def run():
    if OP == "fd":
        pr.dm.numeric_gradient(pr.v, pr.model, pr.b, EPS, g=g)
    elif OP == "energy":
        pr.dm.energy(pr.v, pr.model, pr.b, out=J)
        g[:3] = J
    else:
        pr.dm.exact_gradient(pr.v, pr.model, pr.b, g=g, J=J)
for _ in range(5):
    run()
pr.dm.check()
torch.cuda.synchronize()
n = %d
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
for a, z in ev:
    a.record(); z.record()
A, Z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
A.record()
for a, z in ev:
    pr.dm.time_next(a, z)
    run()
Z.record()
torch.cuda.synchronize()
kern = sorted(a.elapsed_time(z) for a, z in ev)[n // 2]
step = A.elapsed_time(Z) / n
torch.save(g.cpu(), "/tmp/variant_g_%%s.pt" %% %r)
print(json.dumps({"step_ms": step, "kernel_ms": kern, "J": float(J[0]),
                  "cross": pr.dm.stats["cross_entries"], "ctas": pr.dm.stats["ctas_per_sm"]}))
'''


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--n", type=int, default=50)
    ap.add_argument("--op", default="exact", choices=["exact", "fd", "energy"])
    ap.add_argument("variants", nargs="+")
    args = ap.parse_args()
    import json
    res = []
    for k, spec in enumerate(args.variants):
        name, _, envs = spec.partition(":")
        name = name.split("=", 1)[1] if "=" in name else name
        env = dict(os.environ)
        if name != "product":
            env["FM_LIB_OVERRIDE"] = os.path.join(ROOT, "paper_2109_01158_b200", "lib",
                                                  f"libfemmin_{name}.so")
        for kv in filter(None, envs.split(";")):
            a, b = kv.split("=", 1)
            env[a] = b
        tag = str(k)
        code = CHILD % (ROOT, args.config, args.op, args.n if args.op != "fd" else 10, tag)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        if r.returncode:
            print(f"{spec}: FAILED {r.stderr[-400:]}", flush=True)
            continue
        d = json.loads(r.stdout.strip().splitlines()[-1])
        res.append((spec, d, tag))
        print(f"{spec:40s} step {d['step_ms']:.4f} ms  kernel {d['kernel_ms']:.4f} ms  "
              f"cross {d['cross']}  J {d['J']:.12e}", flush=True)
    if len(res) > 1:
        import torch
        g0 = torch.load(f"/tmp/variant_g_{res[0][2]}.pt")
        for spec, d, tag in res[1:]:
            g = torch.load(f"/tmp/variant_g_{tag}.pt")
            print(f"{spec}: max|dg|/max|g| vs first = "
                  f"{float((g - g0).abs().max() / g0.abs().max()):.2e}")


if __name__ == "__main__":
    main()
