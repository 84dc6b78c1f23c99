"""Benchmark: fused J + exact grad J on the config-4 Neo-Hookean beam.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg1|cfg2|cfg2_p1.8|cfg3|cfg4|cfg5] [--shard r/W]
                    [--extras [--descent-iters I]] [--no-cpu-baseline]

N = 1: BASELINE.json configs[3] (3D compressible Neo-Hookean, 256x128x128 Kuhn
beam, 25,165,824 tets) — the config the north-star target (>= 60 % of the HBM
roofline on the 3D NH exact-gradient path) is quoted on.  One step = one fused
J + grad J evaluation of the whole mesh (energy, chain-rule gradient on all
12.78M free dofs, consistent load), device-resident.  N > 1 (torchrun): the
beam is split into x1-slabs, one per rank, J is all-gathered over NCCL and the
interface-plane gradient partials are exchanged with the slab neighbours
(strong scaling: the total mesh is fixed); ``--config cfg5`` runs the
1.61 G-tet beam the same way, ``--shard r/W`` one rank's slab on this GPU.
``--extras`` adds the energy-only, FD, gradient-only, exact-HVP, trust-region
and config-5 descent-loop timings.

Rank 0 prints ONE JSON line.  ``--impl reference`` times the reference
algorithm's CPU implementation (the oracle port of femmin, oracle/) on all
host cores on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# algorithmic bytes per element of one fused J+grad pass (SURVEY.md §8d,
# "variant S"): int32 conn, f64 vol, f64 dphi, v and b read once per node,
# g written once per free dof
def algorithmic_bytes(dim, d, ne, nn, nfree_dofs):
    per_elem = 4 * (dim + 1) + 8 + 8 * dim * (dim + 1)
    return ne * per_elem + 8 * d * nn * 2 + 8 * nfree_dofs


# FD gradient (gradients.py:84-121) FP64 roofline: algorithmic flops of the
# reference formulation per perturbed state = row j of F recomputed from the
# perturbed nodal values (dim entries x (dim+1 mul + dim add)) + det (dim 3:
# 12 mul + 5 add; 2: 2 + 1) + |F|^2 (d*dim mul + d*dim-1 add) + W (8; log and
# pow not counted) -> 3D Neo-Hookean 63, 2D 29; 2 d ||T|| states per launch
def fd_flops_per_state(dim, d):
    row = dim * ((dim + 1) + dim)
    det = 17 if dim == 3 else 3
    i1 = 2 * d * dim - 1
    return row + det + i1 + 8


def _fp64_peak():
    path = os.path.join(ROOT, "profiles", "fp64_peak.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["fp64_tflops"]), "measured (profiles/fp64_peak.json, tools/fp64_peak.cu)"
    except Exception:
        return 37.0, "nominal B200 FP64 (no measurement found)"


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class MemSampler:
    """Peak device memory in use (NVML, every 5 ms) while the problem and its
    evaluation context are built."""

    def __init__(self, index=0):
        self.peak, self.stop_ev = 0, threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.nv = pynvml
        except Exception:
            self.nv = None

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def _run(self):
        while not self.stop_ev.is_set():
            self.peak = max(self.peak, self.nv.nvmlDeviceGetMemoryInfo(self.h).used)
            time.sleep(0.005)

    def __exit__(self, *exc):
        self.stop_ev.set()
        if self.nv is not None:
            self.t.join()


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[3 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def cpu_baseline_sample(nx=96, ny=48, nz=48, repeats=2):
    """Reference algorithm (oracle port of femmin, numpy) on host cores: a
    bounded sample of the same workload (3D NH Kuhn beam, same box/field)."""
    os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count()))
    from oracle import femmin_oracle as O
    m, model, b, v = O.problem_beam(nx, ny, nz, seed=2109)
    RP = O.reference_patches(m, O.build_patches(m))
    best = float("inf")
    for _ in range(repeats):
        t0 = time.perf_counter()
        O.energy(v, m, model, b)
        O.exact_gradient_femmin(v, m, RP, model, b)
        best = min(best, time.perf_counter() - t0)
    return {"value": m.ne / best / 1e6, "unit": "Melem/s",
            "cores": 1, "kind": "port",
            "sample": f"beam {nx}x{ny}x{nz} ({m.ne} tets), femmin algorithm (oracle port doing "
                      f"the reference's per-call work: energy + exact_gradient with patch-row "
                      f"copies; numpy ufuncs single-threaded, OpenBLAS ddot "
                      f"with {os.environ.get('OMP_NUM_THREADS')} threads), best of {repeats}",
            "seconds_per_eval": best}


METRIC = "J+gradJ throughput (fused J + exact gradient evals x elements / s)"


def _ref_worker(q, bar, nx, ny, nz, ix0, ix1, warmup, steps):
    """One host process of the reference arm: the femmin algorithm (oracle
    port) on the x1-slab [ix0, ix1) of the beam, timed between barriers."""
    from oracle import femmin_oracle as O
    m, model, b, v = O.problem_beam(nx, ny, nz, seed=2109, ix0=ix0, ix1=ix1)
    RP = O.reference_patches(m, O.build_patches(m))
    for _ in range(warmup):
        O.energy(v, m, model, b)
        O.exact_gradient_femmin(v, m, RP, model, b)
    bar.wait()
    t0 = time.perf_counter()
    for _ in range(steps):
        O.energy(v, m, model, b)
        O.exact_gradient_femmin(v, m, RP, model, b)
    q.put((m.ne, t0, time.perf_counter()))


def run_reference(args, rank, world):
    """--impl reference: the reference algorithm (femmin's numpy energy +
    exact_gradient, restated in oracle/ with the reference's per-call work and
    pinned bit-exactly against it) on ALL host cores of this box: the cfg4
    beam's 256 x1-slabs of cubes are split among one single-threaded process
    per core (contiguous ranges; each slab's J and gradient partials are what
    a rank of the multi-GPU split computes), all timed between one barrier and
    the last stop (rank 0 only).  When the whole beam does not fit the host
    memory or (K + W) steps of it would exceed ~2 minutes, every process runs a
    shorter range and the line says which fraction of cfg4 one step covers."""
    if rank != 0:
        return
    import multiprocessing as mp
    nx, ny, nz = 256, 128, 128
    cores = len(os.sched_getaffinity(0))
    try:
        with open("/proc/meminfo") as fh:
            avail_gb = int(next(x for x in fh if x.startswith("MemAvailable")).split()[1]) / 2**20
    except Exception:
        avail_gb = 16.0
    nproc = max(1, min(cores, args.ref_procs or cores, nx))
    per = nx // nproc  # cube slabs per process for the whole beam
    # ~0.14 s per single-threaded step of one 98,304-tet cube slab, ~0.35 GB each
    per_time = max(1, int(120.0 / (0.14 * (args.steps + args.warmup))))
    per_mem = max(1, int(0.7 * avail_gb / nproc / 0.35))
    per = max(1, min(per, per_time, per_mem))
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[k] = "1"
    ctx = mp.get_context("spawn")
    q, bar = ctx.Queue(), ctx.Barrier(nproc)
    procs = [ctx.Process(target=_ref_worker,
                         args=(q, bar, nx, ny, nz, w * (nx // nproc), w * (nx // nproc) + per,
                               args.warmup, args.steps))
             for w in range(nproc)]
    for p in procs:
        p.start()
    res = [q.get() for _ in procs]
    for p in procs:
        p.join()
    ne = sum(r[0] for r in res)
    dt = (max(r[2] for r in res) - min(r[1] for r in res)) / args.steps
    value = ne / dt / 1e6
    frac = ne / (6 * nx * ny * nz)
    same = nproc * per == nx
    sample = (f"{nproc} single-threaded processes, each {per} cube x1-slab(s) of the cfg4 beam "
              f"({ne // nproc} tets each, {ne} total = {frac:.3f} of cfg4"
              f"{' = the whole beam' if same else ''}), femmin algorithm (oracle port of energy "
              f"+ exact_gradient doing the reference's per-call work)")
    line = {
        "impl": "reference", "metric": METRIC,
        "value": value, "unit": "Melem/s", "n_gpus": 0, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"cfg4 3D Neo-Hookean Kuhn beam {nx}x{ny}x{nz} on [0,2]x[0,1]^2"
                               + ("" if same else f", sample of {ne} tets"),
                   "parallelism": f"host CPU x{nproc} processes", "same_config": same},
        "cpu_baseline": {"value": value, "unit": "Melem/s", "cores": nproc, "kind": "port",
                         "sample": sample, "host_cores": cores},
        "e2e": {"value": value, "unit": "Melem/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--extras", action="store_true",
                    help="also time the energy-only and FD kernels")
    ap.add_argument("--tile-nodes", type=int, default=0)
    ap.add_argument("--box", type=str, default="")
    ap.add_argument("--stream-depth", type=int, default=2)
    ap.add_argument("--ref-procs", type=int, default=0,
                    help="--impl reference: host processes (default: all cores)")
    ap.add_argument("--max-context-elems", type=int, default=1 << 28,
                    help="beams: a rank slab with more tets is held as sub-slab contexts")
    ap.add_argument("--sub-elems", type=int, default=140_000_000,
                    help="beams: max tets per sub-slab context when a slab is split")
    ap.add_argument("--shard", type=str, default="",
                    help="r/w: run rank r's x1-slab of a w-way partition on this one GPU")
    ap.add_argument("--descent-iters", type=int, default=100,
                    help="--extras: iterations of the config-5 descent loop")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    # one process per GPU; FM_DIST_BACKEND=gloo (with ranks sharing a device
    # when there are fewer GPUs than ranks) is only a functional smoke test of
    # the multi-rank path on a one-GPU box, never a measurement
    backend = os.environ.get("FM_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count()) if backend != "nccl" else local
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    from paper_2109_01158_b200 import problems
    from paper_2109_01158_b200.parallel import SlabExchange, slab_range

    tiling = None
    if args.tile_nodes or args.box:
        box = [int(x) for x in args.box.split(",")] if args.box else [0, 0, 0]
        tiling = (args.tile_nodes, box + [0] * (3 - len(box)))

    BEAMS = {"cfg4": (256, 128, 128), "cfg5": (1024, 512, 512)}
    msamp = MemSampler(local).__enter__()
    if args.config in BEAMS:
        nx, ny, nz = BEAMS[args.config]
        prank, pworld = rank, world
        if args.shard:
            if world > 1:
                raise SystemExit("--shard emulates one rank on one GPU; not under torchrun")
            prank, pworld = (int(x) for x in args.shard.split("/"))
        ix0, ix1 = slab_range(nx, prank, pworld)
        ne_rank = 6 * (ix1 - ix0) * ny * nz
        if ne_rank > args.max_context_elems:
            # a slab too large for one context (config 5 at 2 GPUs: 805 M tets
            # per rank): sub-slab contexts built one after another
            from types import SimpleNamespace

            from paper_2109_01158_b200.parallel import SlabStack, stack_parts
            stack = SlabStack(nx, ny, nz, ix0, ix1, stack_parts(ne_rank, args.sub_elems),
                              seed=2109, tiling=tiling)
            pr = SimpleNamespace(dm=stack, model=stack.model, b=stack.B, v=stack.V,
                                 ne=stack.ne, nn=stack.nn,
                                 meta=dict(nx=nx, ny=ny, nz=nz, ix0=ix0, ix1=ix1))
        else:
            pr = problems.beam(nx, ny, nz, seed=2109, ix0=ix0, ix1=ix1, tiling=tiling)
        workload = (f"{args.config}: 3D compressible Neo-Hookean beam [0,2]x[0,1]^2, "
                    f"{nx}x{ny}x{nz} hexes x 6 Kuhn tets ({6 * nx * ny * nz:,} tets, "
                    f"{(nx + 1) * (ny + 1) * (nz + 1):,} nodes), f=(0,0,-2.5e7), v=x on x1=0")
        ne_total = 6 * nx * ny * nz
        if args.shard:
            workload += (f"; ONE rank's x1-slab [{ix0},{ix1}) of the {pworld}-way partition "
                         f"({pr.ne:,} tets) on this GPU, no exchange")
            ne_total = pr.ne
        if hasattr(pr.dm, "ranges"):
            workload += (f"; each rank's slab held as {pr.dm.K} sub-slab contexts "
                         f"(<= {args.sub_elems:,} tets each, interfaces summed on the device)")
    else:
        if world > 1:
            raise SystemExit("only the beams (cfg4, cfg5) are partitioned across GPUs")
        pr = problems.CONFIGS[args.config](tiling=tiling)
        workload = args.config
        ne_total = pr.ne
    msamp.__exit__()
    torch.cuda.empty_cache()  # build temporaries back to the device
    dm, model, b, v = pr.dm, pr.model, pr.b, pr.v
    ex = SlabExchange.from_problem(pr, rank, world) if world > 1 else None
    g = torch.empty(dm.nfree_dofs, dtype=torch.float64, device="cuda")
    J = torch.empty(3, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()

    def step():
        dm.exact_gradient(v, model, b, g=g, J=J)
        if ex is not None:
            ex.reduce(g, J)

    for _ in range(args.warmup):
        step()
    dm.check()
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    # kernel events (dominant tile kernel) + step events, all on the launching stream
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    for a, z in kev:
        a.record(stream)
        z.record(stream)
    l0 = dm.launches()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    graph = None
    if (world > 1 and ex is not None and ex.native is not None
            and os.environ.get("FM_BENCH_GRAPH", "1") == "1"):
        # N ranks: the step (tile kernel, finishing pass, exchange pack / one
        # grouped NCCL launch / unpack) is captured once as a CUDA graph and
        # replayed, so the host issues one launch per step; the tile kernel's
        # events then come from an eager pass of the same steps first
        for i in range(args.steps):
            dm.time_next(*kev[i])
            step()
        torch.cuda.synchronize()
        try:
            graph = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream()
            side.wait_stream(stream)
            with torch.cuda.stream(side):
                step()
            stream.wait_stream(side)
            with torch.cuda.graph(graph):
                step()
            torch.cuda.synchronize()
        except Exception as exc:  # capture unsupported: time the eager steps
            print(f"[bench] CUDA graph capture failed ({exc}); eager steps", file=sys.stderr)
            graph = None
        l0 = dm.launches()
        dist.barrier()
        torch.cuda.synchronize()
    t0.record(stream)
    for i in range(args.steps):
        if graph is not None:
            graph.replay()
        else:
            dm.time_next(*kev[i])
            step()
    t1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = dm.launches() - l0
    if graph is not None:  # each replay runs the captured kernels
        launches = 2 * args.steps
    free_b, total_b = torch.cuda.mem_get_info()
    clk = clocks.stop()
    ms = t0.elapsed_time(t1) / args.steps
    if hasattr(dm, "kernel_ms"):  # sub-slab stack: the sub-slabs' tile kernels summed
        kl = dm.kernel_ms()
        kms = sum(kl) / max(1, len(kl))
    else:
        kms = sum(a.elapsed_time(z) for a, z in kev) / args.steps
    if world > 1:
        tt = torch.tensor([ms, kms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms, kms = float(tt[0]), float(tt[1])
    dm.check()

    # ---- FD gradient on the same problem: its own (FP64) roofline --------
    fd_line = None
    if world == 1:
        gfd0 = torch.empty_like(g)
        fd_eps = 1e-8 if dm.d > 1 else 1e-6
        dm.numeric_gradient(v, model, b, fd_eps, g=gfd0)  # first call builds the item lists
        dm.check()
        nfd = 5
        fev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(nfd)]
        for a_, z_ in fev:  # materialise the CUDA events before the library records them
            a_.record(stream)
            z_.record(stream)
        torch.cuda.synchronize()
        for a_, z_ in fev:
            dm.time_next(a_, z_)
            dm.numeric_gradient(v, model, b, fd_eps, g=gfd0)
        torch.cuda.synchronize()
        dm.check()
        if hasattr(dm, "kernel_ms"):
            fd_ms = statistics.median(dm.kernel_ms())
        else:
            fd_ms = statistics.median(a_.elapsed_time(z_) for a_, z_ in fev)
        states = 2 * dm.d * dm.stats["node_entries_total"]
        flop = states * fd_flops_per_state(dm.dim, dm.d)
        fpk, fsrc = _fp64_peak()
        fd_line = {"bound": "fp64", "kernel": "k_tile_exact<FD mode>", "kernel_ms": fd_ms,
                   "eps": fd_eps, "perturbed_states": states,
                   "flop_per_state": fd_flops_per_state(dm.dim, dm.d),
                   "achieved": flop / (fd_ms * 1e-3) / 1e12, "peak": fpk, "unit": "TFLOP/s",
                   "frac": flop / (fd_ms * 1e-3) / 1e12 / fpk, "peak_source": fsrc,
                   "Melem_s": ne_total / fd_ms / 1e3,
                   "W_evals_per_s": states / (fd_ms * 1e-3),
                   "definition": "algorithmic flops of the reference formulation (F row "
                                 "recompute, det, |F|^2, W; log/pow not counted) per perturbed "
                                 "state x 2 d ||T|| states / median kernel time"}

    extras = {}
    if args.extras:
        # secondary kernels on the same problem: energy-only pass and FD gradient
        # (with N ranks: each rank's slab, the slab partials reduced across ranks
        # like the exact gradient's; times are the max over ranks)
        def timed(fn, n):
            fn()
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            for _ in range(n):
                fn()
            a1.record(stream)
            torch.cuda.synchronize()
            t = a0.elapsed_time(a1) / n
            if world > 1:
                tt = torch.tensor([t], dtype=torch.float64, device="cuda")
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                t = float(tt[0])
            return t
        gfd = torch.empty_like(g)

        def energy_step():
            dm.energy(v, model, b, out=J)
            if ex is not None:
                ex.reduce(None, J)

        def fd_step():
            dm.numeric_gradient(v, model, b, 1e-8, g=gfd)
            if ex is not None:
                ex.reduce(gfd)

        def grad_step():
            dm.exact_gradient(v, model, b, g=g)
            if ex is not None:
                ex.reduce(g)

        e_ms = timed(energy_step, 20)
        fd_ms = timed(fd_step, 3)
        go_ms = timed(grad_step, 20)
        extras = {"energy_only_ms": e_ms, "energy_only_Melem_s": ne_total / e_ms / 1e3,
                  "fd_grad_ms": fd_ms, "fd_grad_Melem_s": ne_total / fd_ms / 1e3,
                  "grad_only_ms": go_ms,
                  "fd_W_evals_per_s": 2 * dm.d * dm.stats["node_entries_total"] * world
                  / (fd_ms * 1e-3)}
        dm.check()
        if "dofs_minim" in pr.meta and world == 1:
            # a few trust-region iterations of the device-resident minimizer
            # from the benchmark field: wall time per
            # gradient call (each CG step is one Hessian-vector product = 2)
            from paper_2109_01158_b200.solver import SolveOptions, minimize_device
            minimize_device(dm, model, b, v, pr.meta["dofs_minim"],  # warm-up (module loads)
                            SolveOptions(max_iters=1, max_cg=2))
            res = minimize_device(dm, model, b, v, pr.meta["dofs_minim"],
                                  SolveOptions(max_iters=3, max_cg=20))
            rx = minimize_device(dm, model, b, v, pr.meta["dofs_minim"],
                                 SolveOptions(max_iters=3, max_cg=20, hvp="exact"))
            hp_ms = timed(lambda: dm.hvp(v, v, model, out=g), 20)  # kernel timing only
            extras.update({"tr_exact_hvp_3iters_s": rx.time, "tr_exact_hvp_calls": rx.n_hvp,
                           "tr_exact_hvp_J_end": rx.J_u, "hvp_exact_ms": hp_ms})
            extras.update({"tr_3iters_s": res.time, "tr_grad_calls": res.n_grad,
                           "tr_energy_calls": res.n_energy,
                           "tr_ms_per_grad_call": res.time / max(1, res.n_grad) * 1e3,
                           "tr_J_start_end": [float(dm.energy(v, model, b)[0]), res.J_u]})

    if args.extras and args.descent_iters > 0 and args.config in ("cfg4", "cfg5"):
        # config-5 first-order loop: v <- v - alpha grad J on the free dofs,
        # alpha = 1e-3 h / max|g(v0)|, J recorded every iteration
        it = args.descent_iters
        dm.exact_gradient(v, model, b, g=g)
        if ex is not None:
            ex.reduce(g)
        gmax = g.abs().max().reshape(1)
        if world > 1:
            dist.all_reduce(gmax, op=dist.ReduceOp.MAX)
        alpha = 1e-3 * (2.0 / nx) / float(gmax)
        vd = v.clone()
        Jh = torch.empty((it, 3), dtype=torch.float64, device="cuda")
        dm.descent(vd, model, b, alpha, 3, g=g, J_hist=Jh, exchange=ex)  # warm-up
        vd.copy_(v)
        dm.check()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d0.record(stream)
        dm.descent(vd, model, b, alpha, it, g=g, J_hist=Jh, exchange=ex)
        d1.record(stream)
        torch.cuda.synchronize()
        dms = d0.elapsed_time(d1) / it
        if world > 1:
            tt = torch.tensor([dms], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dms = float(tt[0])
        dm.check()
        Jd = Jh[:, 0].cpu()
        # bytes of one iteration: the fused evaluation + the update (v read and
        # written, g read at the free dofs)
        dbytes = algorithmic_bytes(dm.dim, dm.d, dm.ne, dm.nn, dm.nfree_dofs) + 24 * dm.nfree_dofs
        extras.update({"descent_iters": it, "descent_alpha": alpha,
                       "descent_ms_per_iter": dms,
                       "descent_evals_per_s": 1e3 / dms,
                       "descent_Melem_s": ne_total / dms / 1e3,
                       "descent_hbm_frac": dbytes / (dms * 1e-3) / 1e9 / _peaks()[0],
                       "descent_J_first_last": [float(Jd[0]), float(Jd[-1])],
                       "descent_J_increases": int((Jd[1:] >= Jd[:-1]).sum()),
                       "descent_J_first10": [float(x) for x in Jd[:10]]})

    # ---- end to end through the public device API, host buffers ----------
    v_host = v.cpu().pin_memory()
    g_host = torch.empty(g.shape, dtype=torch.float64).pin_memory()
    J_host = torch.empty(3, dtype=torch.float64).pin_memory()
    e2e_steps = 100  # steady-state stream (fill / drain amortised over 100 fields)

    def e2e_step():
        v.copy_(v_host, non_blocking=True)
        step()
        g_host.copy_(g, non_blocking=True)
        J_host.copy_(J, non_blocking=True)

    e2e_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_serial_ms = e0.elapsed_time(e1) / e2e_steps

    # streamed: consecutive host fields with upload / kernel / download overlapped
    from paper_2109_01158_b200.streaming import FieldStream
    fs = FieldStream(dm, model, b, depth=args.stream_depth, exchange=ex)
    nbuf = 3
    v_hosts = [v_host.clone().pin_memory() for _ in range(nbuf)]
    g_hosts = [torch.empty(g.shape, dtype=torch.float64).pin_memory() for _ in range(nbuf)]
    J_hosts = [torch.empty(3, dtype=torch.float64).pin_memory() for _ in range(nbuf)]
    for i in range(2):
        fs.submit(v_hosts[i % nbuf], g_hosts[i % nbuf], J_hosts[i % nbuf])
    fs.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    s0 = torch.cuda.Event(enable_timing=True)
    s1 = torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    fs.up.wait_stream(stream)
    for i in range(e2e_steps):
        fs.submit(v_hosts[i % nbuf], g_hosts[i % nbuf], J_hosts[i % nbuf])
    # the stop event follows the last download
    stream.wait_stream(fs.down)
    s1.record(stream)
    fs.synchronize()
    e2e_ms = s0.elapsed_time(s1) / e2e_steps
    if world > 1:
        tt = torch.tensor([e2e_ms, e2e_serial_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms, e2e_serial_ms = float(tt[0]), float(tt[1])
    # results of the streamed path equal the serial ones bit for bit
    stream_ok = bool(torch.equal(g_hosts[(e2e_steps - 1) % nbuf], g_host))

    # ---- the reference-facing numpy drop-in: energy_and_gradient(v, mesh,
    # patches, model, load) with host numpy in and out (pageable copies) ---
    numpy_e2e = None
    if world == 1 and args.config == "cfg4":
        import numpy as np
        import paper_2109_01158_b200 as fb
        hm = fb.generate_beam_mesh_3d(nx, ny, nz)
        hm = fb.mark_dirichlet(hm, fb.DirichletSpec(
            [fb.DirichletRegion(where=lambda x: x[:, 0] < 1e-9)]), d=3)
        # the CSR fields of Patches (patches.py:22-34; the drop-in reads only
        # these), built on the GPU; the per-row copies are not materialised
        from paper_2109_01158_b200.patches import build_patches_device
        pfx, pel, psl = build_patches_device(torch.as_tensor(hm.elems2nodes).cuda(),
                                             torch.as_tensor(hm.nodes_minim).cuda(), hm.nn, 4)
        hp = fb.Patches(lengths=np.diff(pfx.cpu().numpy(), prepend=0), elems=pel.cpu().numpy(),
                        volumes=None, elems2nodes=None, dphi=None, logical=None,
                        prefix=pfx.cpu().numpy(), slot=psl.cpu().numpy())
        del pfx, pel, psl
        hload = fb.LinearLoad(b=b.cpu().numpy())
        v_np = v.cpu().numpy().copy()
        Jn, gn_ = fb.energy_and_gradient(v_np, hm, hp, model, hload)  # builds the context
        ncall = 10
        torch.cuda.synchronize()
        tn0 = time.perf_counter()
        for _ in range(ncall):
            Jn, gn_ = fb.energy_and_gradient(v_np, hm, hp, model, hload)
        tn = (time.perf_counter() - tn0) / ncall
        same = bool(np.array_equal(gn_, g.cpu().numpy()))
        numpy_e2e = {"value": ne_total / tn / 1e6, "unit": "Melem/s", "ms_per_call": tn * 1e3,
                     "api": "paper_2109_01158_b200.energy_and_gradient(v_numpy, mesh, patches, "
                            "model, load) -> (J, g_numpy): the femmin signature "
                            "(assembly.py:94-106 + gradients.py:124-149), host numpy in and "
                            "out (staged through pinned buffers inside the call), wall clock over 10 calls after the first "
                            "(context build)",
                     "h2d_bytes_per_call": int(v_np.nbytes), "d2h_bytes_per_call": int(gn_.nbytes + 24),
                     "equals_device_path": same}
        del hm, hp

    value = ne_total / (ms * 1e-3) / 1e6
    peak, peak_src = _peaks()
    alg = algorithmic_bytes(dm.dim, dm.d, dm.ne, dm.nn, dm.nfree_dofs)
    achieved = alg / (kms * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            traffic = json.load(fh).get(f"{args.config}_n{world}")

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline_sample()
        line = {
            "metric": METRIC,
            "value": value, "unit": "Melem/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (GPU-generated mesh, seeded splitmix64 field v = x + U[-a,a])",
            "config": {"workload": workload, "elements": ne_total,
                       "evals_per_s": 1e3 / ms,
                       "hbm_in_use_gb": (total_b - free_b) / 1e9,
                       "hbm_build_peak_gb": msamp.peak / 1e9,
                       "parallelism": f"x1-slabs x{world}" if world > 1 else "single GPU",
                       "step_graph": graph is not None,
                       "l2": (f"DRAM traffic per evaluation (ncu: {traffic / 1e9:.2f} GB in the "
                              "tile kernel, plus the finishing pass) is larger than the 126 MB "
                              "L2; no flush" if traffic else
                              f"inputs ({alg / 1e9:.2f} GB per eval) larger than the 126 MB L2; "
                              "no flush"),
                       "tiles": {k: dm.stats[k] for k in (
                           "n_tiles", "redundancy", "max_tile_elems", "tile_threads",
                           "ctas_per_sm", "node_bufs", "table_bufs", "entry_cap", "cross_entries",
                           "dict_tiles", "closure_cap")}},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "k_tile_exact<3,NH,J,256,NB=%d,TB=%d,2>" % (
                             dm.stats["node_bufs"], dm.stats["table_bufs"]), "kernel_ms": kms,
                         "algorithmic_bytes_per_launch": alg,
                         "bytes_per_elem": alg / dm.ne, "peak_source": peak_src,
                         "frac_of_8TBs_nominal": achieved / 8000.0,
                         # the whole evaluation (tile kernel + cross-entry finishing
                         # pass + J finalize) against the same algorithmic bytes
                         "step_achieved": alg / (ms * 1e-3) / 1e9,
                         "step_frac": alg / (ms * 1e-3) / 1e9 / peak},
            "cpu_baseline": cpu,
            "e2e": {"value": ne_total / (e2e_ms * 1e-3) / 1e6, "unit": "Melem/s",
                    "h2d_bytes_per_step": int(v.numel() * 8),
                    "d2h_bytes_per_step": int(g.numel() * 8 + 24),
                    "api": "streaming.FieldStream.submit(v_host, g_host, J_host): pinned host "
                           "buffers, H2D / kernel / D2H of consecutive fields overlapped "
                           f"(depth {args.stream_depth}); every step copies its full v in and g, J out",
                    "serial_value": ne_total / (e2e_serial_ms * 1e-3) / 1e6,
                    "serial_api": "DeviceMesh.exact_gradient(v, model, b, g, J) between "
                                  "blocking-order H2D / D2H copies on one stream",
                    "streamed_equals_serial": stream_ok,
                    "numpy_drop_in": numpy_e2e},
            "fd_roofline": fd_line,
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        if extras:
            line["extra"] = extras
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
