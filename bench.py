"""bench.py -- BC-preconditioned GMRES time-to-tol on B200 (BASELINE.json metric).

Headline (N=1): BASELINE configs[2], the largest configuration that fits one GPU's role in the
BASELINE list (config 3 is specified as the 8-GPU case): 2D Riesz FDE, gamma 1.3/1.7,
255^2 x 512 = 33.3 M DoF, GMRES(20) right-preconditioned with the BC preconditioner, tol 1e-10,
fp64, seeded uniform source.  A "step" = one full solve with b resident in HBM: the reference's
timed span krylov.hpp:87-190 (k+1 PC applies, k+1 matvecs, the Gram-Schmidt work, x = P^{-1} V y
and the fresh TRR).  Configs 1 (1D 8191 x 2048, gamma 1.2) and 3 (2D 1023^2 x 1024, GMRES(10),
tol 1e-9) are measured after it in the same run and reported under "secondary".

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 2]
  python bench.py --sweep [--sweep-nx 1023,65535] [--sweep-nt 256,8192]   (config 4, one line per point)

N > 1 (torchrun): ONE solve sharded over the N ranks (paper_2003_07020_b200/distributed.py:
time-sharded Krylov vectors, NCCL all-to-all around the tau solves, all-reduce for the dots;
scaling "strong"); --replicas instead runs N independent solves (scaling "weak").
--impl reference times the reference's own CPU solver (oracle/_ref: the unmodified reference
headers compiled by oracle/Makefile) on this host's cores: one full, unextrapolated solve per step.
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "BC-preconditioned GMRES time-to-tol (solves/s)"
UNIT = "solves/s"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device, self.rows, self.proc = device, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        return False

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------------------------ reference arm
def ref_problem(w):
    """The unmodified reference (oracle/_ref) on workload w, plan built (driver.hpp:49-73)."""
    from oracle import oracle as O
    ref = O.Reference()
    if w.two_dim:
        p = ref.problem_2d(w.gamma[0], w.gamma[1], 1.0, 1.0, w.h, w.n, w.n_time, w.dt).build_plan()
    else:
        p = ref.problem_1d(w.gamma[0], 1.0, w.h, w.n, w.n_time, w.dt).build_plan()
    return ref, p


def cpu_reference_solve(w, threads: int):
    """ONE full reference solve (gmres_right as driver.hpp:62-73 wires it; GMRES(m) through the
    restart emulation of SURVEY §8(c) when the solve needs more than m steps).  Returns
    (seconds of the reference's own timed span krylov.hpp:87-190, iterations)."""
    from paper_2003_07020_b200 import problems
    ref, p = ref_problem(w)
    ref.set_threads(threads)
    b = problems.rhs(w)
    _, rep = p.gmres(b, w.tol, 200)
    if rep.iterations > w.restart > 0:  # GMRES(m) differs from the unrestarted solve: emulate it
        _, r2 = p.gmres_restarted(b, w.tol, 200, w.restart)
        return r2["seconds"], r2["iterations"]
    return rep.seconds, rep.iterations


def cpu_reference_ops(w, threads: int):
    """The reference's apply_inverse and AllAtOnceOperator::apply, one call each, wall-clock."""
    from paper_2003_07020_b200 import problems
    ref, p = ref_problem(w)
    ref.set_threads(threads)
    b = problems.rhs(w)
    t0 = time.perf_counter()
    p.pc_apply(b)
    t1 = time.perf_counter()
    p.matvec(b)
    t2 = time.perf_counter()
    return t1 - t0, t2 - t1


def run_reference(args, w):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    # K timed full solves behind W untimed ones, like the GPU arm; every step is one complete reference
    # solve (nothing extrapolated).  A wall-clock budget guards the driver's limit on a slow host: warm-up
    # solves are dropped first, then timed ones, and the line reports what actually ran.
    budget = float(os.environ.get("FPC_REF_BUDGET_S", "1300"))
    t_start = time.perf_counter()
    want_k, want_w = args.steps_ref, args.warmup_ref
    times, iters, warm, est = [], None, 0, None
    reserve = 0.0  # the single-thread / nproc operator timings after the solves (~1.3 solves' worth at config 2)
    while len(times) < want_k:
        elapsed = time.perf_counter() - t_start
        if est is not None:
            reserve = 1.5 * est
            left = budget - elapsed - reserve
            if warm < want_w and left < (want_k + 1) * est:
                want_w = warm  # no room for another warm-up solve
            if left < est and times:
                break
        sec, iters = cpu_reference_solve(w, threads)
        est = sec if est is None else max(est, sec)
        if warm < want_w:
            warm += 1
        else:
            times.append(sec)
    args.steps_ref, args.warmup_ref = len(times), warm
    t = statistics.mean(times)
    val = 1.0 / t
    # the single-thread figure (set_thread_count(1), parallel.hpp:24) beside nproc: one PC apply and
    # one matvec of the same workload at each thread count (a 1-thread full solve is ~16x longer)
    pc1, mv1 = cpu_reference_ops(w, 1)
    pcn, mvn = cpu_reference_ops(w, threads)
    sample = (f"reference gmres_right (oracle/_ref, unmodified headers) on {w.name}: {args.steps_ref} full solves of "
              f"{iters} iterations ({args.warmup_ref} untimed ones first), {threads} threads, the reference's own report.seconds (krylov.hpp:87-190)")
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world,
            "steps": args.steps_ref, "warmup": args.warmup_ref, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded uniform source)",
            "config": workload_config(w),
            "iterations": iters, "step_seconds": times,
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample,
                             "cpu_model": cpu_model()},
            "single_thread": {"threads": 1, "pc_apply_s": pc1, "matvec_s": mv1,
                              "nproc": {"threads": threads, "pc_apply_s": pcn, "matvec_s": mvn},
                              "note": "one apply_inverse and one AllAtOnceOperator::apply of this workload at "
                                      "set_thread_count(1) and at nproc"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def workload_config(w):
    c = {"workload": w.name, "n_space": w.n_space, "n_time": w.n_time, "dof": w.dim,
         "gamma": list(w.gamma), "kappa": list(w.kappa), "tol": w.tol, "restart": w.restart,
         "solver": f"GMRES({w.restart}) right-preconditioned, BC alpha=min(0.5, dt/2)", "seed": w.seed}
    if w.two_dim:
        c["n_per_dim"] = w.n
    return c


# ------------------------------------------------------------------------------------ sharded
def run_sharded(args, w, rank, world, local):
    """N > 1: ONE config solve frequency-sharded over the N ranks: time-sharded
    Krylov vectors, NCCL all-to-all around the tau solves, all-reduce for the dots."""
    import torch
    import torch.distributed as dist

    import paper_2003_07020_b200 as fp
    from paper_2003_07020_b200 import problems
    from paper_2003_07020_b200.distributed import CudaShardKernels, ShardedSolver
    dev = torch.device("cuda", local)
    ctx = fp.Context(local, torch.cuda.current_stream(dev))
    jac = (fp.RieszJacobian2D(w.gamma[0], w.gamma[1], 1.0, 1.0, w.h, w.n) if w.two_dim
           else fp.RieszJacobian1D(w.gamma[0], 1.0, w.h, w.n))
    op = fp.AllAtOnceOperator(fp.TimeStencil(w.n_time), jac, w.dt, ctx)
    plan = fp.build_plan(fp.PreconditionerKind.generalized(), w.n_time, w.dt, op,
                         ordering=fp.Ordering[args.ordering])
    s = ShardedSolver(w.n_time, w.n_space, CudaShardKernels(op, plan), ordering=args.ordering,
                      transport=args.transport)
    try:
        _run_sharded_timed(args, w, rank, world, local, s, dev, fp, problems)
    finally:
        s.close()
    dist.destroy_process_group()


def _run_sharded_timed(args, w, rank, world, local, s, dev, fp, problems):
    import torch
    import torch.distributed as dist
    b_host = problems.rhs(w)
    lo, hi = s.koff * w.n_space, (s.koff + s.nt_loc) * w.n_space
    b_loc_host = np.ascontiguousarray(b_host[lo:hi])
    b = torch.from_numpy(b_loc_host).to(dev)
    for _ in range(args.warmup):
        x, rep = s.gmres(b, w.tol, 200, w.restart)
    launches0 = fp.kernel_launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        dist.barrier()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(args.steps):
            x, rep = s.gmres(b, w.tol, 200, w.restart)
        e1.record()
        torch.cuda.synchronize()
        dist.barrier()
    t = e0.elapsed_time(e1) * 1e-3 / args.steps
    tt = torch.tensor([t], device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t = float(tt.item())
    launches = fp.kernel_launches() - launches0
    pin = torch.from_numpy(b_loc_host).pin_memory()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        bd = pin.to(dev, non_blocking=True)
        xd, _ = s.gmres(bd, w.tol, 200, w.restart)
        xh = xd.cpu()
    te = (time.perf_counter() - t0) / args.steps
    tt = torch.tensor([te], device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    te = float(tt.item())
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": 1.0 / t, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded uniform[-1,1] source)",
            "config": {"workload": w.name, "n_space": w.n, "n_time": w.n_time, "tol": w.tol, "restart": w.restart,
                       "parallelism": f"frequency-sharded x{world} ("
                                      + ("NCCL all-to-all" if args.transport == "nccl" else "peer-store exchanges")
                                      + " + all-reduce)",
                       "pc_ordering": args.ordering},
            "iterations": rep.iterations, "true_relative_residual": rep.true_relative_residual,
            "e2e": {"value": 1.0 / te, "unit": UNIT, "h2d_bytes_per_step": 8 * (hi - lo),
                    "d2h_bytes_per_step": 8 * (hi - lo)},
            "gpu_launches": launches, "clocks": clk.summary(), "cpu_baseline": None}))


# ------------------------------------------------------------------------------------ config-4 sweep
SWEEP_NX = [1023, 2047, 4095, 8191, 16383, 32767, 65535]
SWEEP_NT = [256, 512, 1024, 2048, 4096, 8192]


def run_sweep(args):
    """BASELINE config 4: isolated BC preconditioner apply + matvec, 1D gamma=1.5, Nx x Nt grid,
    complex128 seeded Gaussian input = a batch of two real vectors (Re, Im) since the operators are
    real-linear; `reps` applications each, device-resident, CUDA events on the
    library stream.  One JSON line per point (not the headline metric)."""
    import torch
    import paper_2003_07020_b200 as fp
    rank, world, local = dist_env()
    if world > 1 or args.sweep_sharded:
        run_sweep_sharded(args, rank, world, local)
        return
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device=dev)
    ctx = fp.Context(0, stream)
    peak, peak_kind = load_peaks()
    nxs = [int(x) for x in args.sweep_nx.split(",")] if args.sweep_nx else SWEEP_NX
    nts = [int(x) for x in args.sweep_nt.split(",")] if args.sweep_nt else SWEEP_NT
    ref = None
    if not args.no_cpu_baseline:
        try:
            from oracle import oracle as O
            ref = O.Reference()
            ref.set_threads(os.cpu_count() or 1)
        except Exception:  # noqa: BLE001
            ref = None
    for nx in nxs:
        for nt in nts:
            h, dt = 1.0 / (nx + 1), 1.0 / nt
            op = fp.AllAtOnceOperator(fp.TimeStencil(nt), fp.RieszJacobian1D(1.5, 1.0, h, nx), dt, ctx)
            plan = fp.build_plan(fp.PreconditionerKind.generalized(), nt, dt, op)
            N = nx * nt
            gen = torch.Generator(device=dev)
            gen.manual_seed(20260819 + nx * 131 + nt)
            with torch.cuda.stream(stream):
                xr = torch.randn(N, dtype=torch.float64, device=dev, generator=gen)
                xi = torch.randn(N, dtype=torch.float64, device=dev, generator=gen)
                yr = torch.empty_like(xr)
                yi = torch.empty_like(xi)
            stream.synchronize()

            def timed(fn, reps):
                for _ in range(args.warmup):
                    fn()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(reps):
                    fn()
                e1.record(stream)
                torch.cuda.synchronize()
                return e0.elapsed_time(e1) * 1e-3 / reps

            def pc():
                fp.apply_inverse(plan, xr, yr)
                fp.apply_inverse(plan, xi, yi)

            def mv():
                op.apply(xr, yr)
                op.apply(xi, yi)

            # torch's current stream = the library stream: the API's cross-stream ordering events
            # (two per call) are not needed and are skipped
            with ClockSampler(0) as clk, torch.cuda.stream(stream):
                t_pc = timed(pc, args.sweep_reps)
                t_mv = timed(mv, args.sweep_reps)
            H = nt // 2 + 1
            B_pc = 2 * (16.0 * N + 64.0 * H * nx)   # SURVEY §8(d), two real vectors per complex input
            B_mv = 2 * 16.0 * N
            cpu = None
            if ref is not None and N <= args.sweep_cpu_max:
                p = ref.problem_1d(1.5, 1.0, h, nx, nt, dt)
                p.build_plan()
                xh = xr.cpu().numpy()
                t0 = time.perf_counter()
                p.pc_apply(xh)
                t_ref = 2 * (time.perf_counter() - t0)
                cpu = {"value": 1.0 / t_ref, "unit": "complex PC applies/s", "cores": os.cpu_count(),
                       "kind": "reference", "sample": "one real apply_inverse of oracle/_ref, x2 for (Re, Im)"}
            line = {"metric": "config-4 sweep: BC PC applies/s and matvecs/s (complex128 input)",
                    "config": {"workload": "cfg4_sweep", "n_space": nx, "n_time": nt, "gamma": 1.5, "reps": args.sweep_reps,
                               "input": "complex128 Gaussian = (Re, Im) real batch of 2"},
                    "pc_applies_per_s": 1.0 / t_pc, "matvecs_per_s": 1.0 / t_mv,
                    "pc_apply_gbs": B_pc / t_pc / 1e9, "matvec_gbs": B_mv / t_mv / 1e9,
                    "pc_apply_hbm_frac": B_pc / t_pc / 1e9 / peak, "matvec_hbm_frac": B_mv / t_mv / 1e9 / peak,
                    "peak_gbs": peak, "peak_source": peak_kind, "l2_resident": 32.0 * N < 100e6,
                    "clocks": clk.summary(), "cpu_baseline": cpu}
            print(json.dumps(line), flush=True)
            del op, plan, xr, xi, yr, yi
            torch.cuda.empty_cache()


def run_sweep_sharded(args, rank, world, local):
    """Config 4 at N > 1 (torchrun): every (Nx, Nt) point's PC apply and matvec run sharded over the
    N ranks (distributed.py ShardedSolver: time-sharded vectors, the four all-to-alls around the
    frequency-sharded tau solves, the BDF2 halo); the same complex128 = (Re, Im) batch of two real
    vectors per application; time = max over ranks of CUDA events on the rank's stream."""
    import torch
    import torch.distributed as dist

    import paper_2003_07020_b200 as fp
    from paper_2003_07020_b200.distributed import CudaShardKernels, ShardedSolver
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", rank=rank, world_size=world)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    ctx = fp.Context(local, torch.cuda.current_stream(dev))
    peak, peak_kind = load_peaks()
    nxs = [int(x) for x in args.sweep_nx.split(",")] if args.sweep_nx else SWEEP_NX
    nts = [int(x) for x in args.sweep_nt.split(",")] if args.sweep_nt else SWEEP_NT
    for nx in nxs:
        for nt in nts:
            if nt % world or nt // world < 2:
                continue
            h, dt = 1.0 / (nx + 1), 1.0 / nt
            op = fp.AllAtOnceOperator(fp.TimeStencil(nt), fp.RieszJacobian1D(1.5, 1.0, h, nx), dt, ctx)
            plan = fp.build_plan(fp.PreconditionerKind.generalized(), nt, dt, op)
            s = ShardedSolver(nt, nx, CudaShardKernels(op, plan), transport=args.transport)
            try:
                gen = torch.Generator(device=dev)
                gen.manual_seed(20260819 + nx * 131 + nt + 7919 * rank)
                nloc = s.nt_loc * nx
                xr = torch.randn(nloc, dtype=torch.float64, device=dev, generator=gen)
                xi = torch.randn(nloc, dtype=torch.float64, device=dev, generator=gen)

                def timed(fn, reps):
                    for _ in range(args.warmup):
                        fn()
                    dist.barrier()
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(reps):
                        fn()
                    e1.record()
                    torch.cuda.synchronize()
                    t = torch.tensor([e0.elapsed_time(e1) * 1e-3 / reps], device=dev)
                    dist.all_reduce(t, op=dist.ReduceOp.MAX)
                    return float(t.item())

                t_pc = timed(lambda: (s.pc_apply(xr), s.pc_apply(xi)), args.sweep_reps)
                t_mv = timed(lambda: (s.matvec(xr), s.matvec(xi)), args.sweep_reps)
            finally:
                s.close()
            N = nx * nt
            H = nt // 2 + 1
            B_pc = 2 * (16.0 * N + 64.0 * H * nx)
            B_mv = 2 * 16.0 * N
            if rank == 0:
                print(json.dumps({
                    "metric": "config-4 sweep: BC PC applies/s and matvecs/s (complex128 input)", "n_gpus": world,
                    "scaling": "strong",
                    "config": {"workload": "cfg4_sweep", "n_space": nx, "n_time": nt, "gamma": 1.5,
                               "reps": args.sweep_reps, "input": "complex128 Gaussian = (Re, Im) real batch of 2",
                               "parallelism": f"time-sharded x{world} ({args.transport} exchanges)"},
                    "pc_applies_per_s": 1.0 / t_pc, "matvecs_per_s": 1.0 / t_mv,
                    "pc_apply_gbs": B_pc / t_pc / 1e9, "matvec_gbs": B_mv / t_mv / 1e9,
                    "pc_apply_hbm_frac_per_gpu": B_pc / t_pc / 1e9 / peak / world,
                    "matvec_hbm_frac_per_gpu": B_mv / t_mv / 1e9 / peak / world,
                    "peak_gbs": peak, "peak_source": peak_kind}), flush=True)
            del op, plan, s
            torch.cuda.empty_cache()
    dist.destroy_process_group()


# ------------------------------------------------------------------------------------ our arm
def load_onchip_peaks():
    """fp64 / shared-memory roofs measured on the B200 by scripts/onchip_peaks.cu (profiles/)."""
    try:
        with open(os.path.join(ROOT, "profiles", "onchip_peaks.json")) as f:
            return json.load(f)
    except Exception:  # noqa: BLE001
        return {}


def fft_flops(w):
    """SURVEY §8(d) algorithmic FLOPs of one matvec (the reference's algorithm: two complex FFTs
    of the circulant length L per Toeplitz product) -- 1D: Nt (5 L log2 L + L) + 6N; 2D: 2n
    Toeplitz products per time level."""
    import math
    N = w.dim
    L = 1 << math.ceil(math.log2(2 * w.n))
    per = 5.0 * L * math.log2(L) + L
    return w.n_time * (2 * w.n if w.two_dim else 1) * per + (8.0 if w.two_dim else 6.0) * N


def solve_bytes(w, k):
    """SURVEY §8(d) compulsory bytes of a k-iteration solve: (k+1)(B_mv + B_pc) + sum_j 8N(2j+5)
    (one Gram-Schmidt pass per step, j counted within a restart cycle) + 8N(k+1) + 16N + per
    restart (B_mv + 24N)."""
    N = w.dim
    H = w.n_time // 2 + 1
    B_mv, B_pc = 16.0 * N, 16.0 * N + 64.0 * H * w.n_space
    rcyc = w.restart if w.restart else k + 1
    n_restarts = max(0, (k - 1) // rcyc) if k > 0 else 0
    return ((k + 1) * (B_mv + B_pc) + sum(8.0 * N * (2 * (j % rcyc) + 5) for j in range(k))
            + 8.0 * N * (k + 1) + 16.0 * N + n_restarts * (B_mv + 24.0 * N)), B_mv, B_pc


def build_ours(fp, w, ctx, ordering="reference"):
    if w.two_dim:
        jac = fp.RieszJacobian2D(w.gamma[0], w.gamma[1], 1.0, 1.0, w.h, w.n)
    else:
        jac = fp.RieszJacobian1D(w.gamma[0], 1.0, w.h, w.n)
    op = fp.AllAtOnceOperator(fp.TimeStencil(w.n_time), jac, w.dt, ctx)
    plan = fp.build_plan(fp.PreconditionerKind.generalized(), w.n_time, w.dt, op, ordering=fp.Ordering[ordering])
    return op, plan


def measure(fp, torch, w, args, stream, ctx, dev, steps, warmup, full, sync=None):
    """Device-resident time-to-tol of w (K solves between events on the library stream), plus,
    when `full`: live per-kernel times, operator rates, the roofline of the dominant kernel and the
    e2e solve through the C-ABI with pinned host buffers."""
    from paper_2003_07020_b200 import problems
    op, plan = build_ours(fp, w, ctx, args.ordering)
    cfg = fp.SolverConfig(tol=w.tol, max_iter=200, restart=w.restart)
    b_host = problems.rhs(w)
    N = w.dim
    with torch.cuda.stream(stream):
        b = torch.from_numpy(b_host).to(dev)
        x = torch.empty_like(b)
    stream.synchronize()
    for _ in range(warmup):
        res = fp.gmres_right(op, plan, b, cfg, out=x)
    torch.cuda.synchronize()
    k = int(res.report.iterations)
    launches0 = fp.kernel_launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clk:
        if sync:
            sync()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(steps):
            res = fp.gmres_right(op, plan, b, cfg, out=x)
        ev1.record(stream)
        torch.cuda.synchronize()
        if sync:
            sync()
    launches = fp.kernel_launches() - launches0
    t_step = ev0.elapsed_time(ev1) * 1e-3 / steps
    out = {"ms_per_step": t_step * 1e3, "value": 1.0 / t_step, "iterations": k, "restarts": int(res.report.restarts),
           "true_relative_residual": res.report.true_relative_residual, "gpu_launches": launches,
           "clocks": clk.summary()}
    B_tot, B_mv, B_pc = solve_bytes(w, k)
    peak, peak_kind = load_peaks()
    out["solve_roofline"] = {"bound": "hbm", "algorithmic_bytes": B_tot, "achieved": B_tot / t_step / 1e9,
                             "peak": peak, "unit": "GB/s", "frac": B_tot / t_step / 1e9 / peak,
                             "formula": "SURVEY 8(d) B_tot, one Gram-Schmidt pass per step (the reference "
                                        "re-orthogonalises every step here, which doubles that term)"}
    if not full:
        with fp.KernelProfile() as prof:  # live per-kernel device time inside one more solve
            fp.gmres_right(op, plan, b, cfg, out=x)
        out["kernel_time_ms_per_solve"] = {k_: v[0] for k_, v in prof.table.items()}
        out["kernel_launches_per_solve"] = {k_: v[1] for k_, v in prof.table.items()}
        del b, x, res, op, plan
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        return out
    x_sample = x[::1009].cpu().numpy()  # checked against the e2e (host-buffer) solve below

    with fp.KernelProfile() as prof:  # live per-kernel device time inside one solve
        fp.gmres_right(op, plan, b, cfg, out=x)
    table = prof.table

    def rate(fn, reps=20):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e-3 / reps

    y = x  # the solution buffer is free again
    t_mv = rate(lambda: op.apply(b, y))
    t_pc = rate(lambda: fp.apply_inverse(plan, b, y))
    H = w.n_time // 2 + 1
    out.update({"pc_applies_per_s": 1.0 / t_pc, "matvecs_per_s": 1.0 / t_mv,
                "pc_apply_gbs": B_pc / t_pc / 1e9, "matvec_gbs": B_mv / t_mv / 1e9})

    # dominant kernel by live device time inside the solve; algorithmic bytes per launch
    dom_name, (dom_ms, dom_cnt) = max(table.items(), key=lambda kv: kv[1][0])
    per_launch_bytes = {"matvec_1d": B_mv, "matvec_2d": B_mv, "time_fwd": 8.0 * N + 16.0 * H * w.n_space,
                        "time_inv": 8.0 * N + 16.0 * H * w.n_space, "tau_solve_1d": 32.0 * H * w.n_space,
                        "tau_solve_2d": 32.0 * H * w.n_space}
    dom_bytes = per_launch_bytes.get(dom_name)
    dom_t = dom_ms * 1e-3 / dom_cnt
    achieved = dom_bytes / dom_t / 1e9 if dom_bytes else None
    traffic = onchip = None
    for fname, key in (("traffic.json", "traffic"), ("onchip.json", "onchip")):
        fpath = os.path.join(ROOT, "profiles", fname)
        if os.path.exists(fpath):
            try:
                val = json.load(open(fpath)).get(w.name, {}).get(dom_name)
            except Exception:  # noqa: BLE001
                val = None
            if key == "traffic":
                traffic = val
            else:
                onchip = val
    roof = {"bound": "hbm", "kernel": dom_name, "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": (achieved / peak) if achieved else None, "traffic": traffic,
            "algorithmic_bytes_per_launch": dom_bytes, "avg_launch_us": dom_t * 1e6, "peak_source": peak_kind,
            "onchip": onchip}
    ocp = load_onchip_peaks()
    if dom_name.startswith("matvec") and ocp.get("fp64_fma_tflops"):
        f = fft_flops(w)
        roof["fp64"] = {"flops_per_launch": f, "achieved_tflops": f / dom_t / 1e12,
                        "peak_tflops": ocp["fp64_fma_tflops"], "frac": f / dom_t / 1e12 / ocp["fp64_fma_tflops"],
                        "formula": "SURVEY 8(d) F_mv (reference algorithm: two complex FFTs of length L per "
                                   "Toeplitz product)", "peak_source": "profiles/onchip_peaks.json (measured)"}
    if onchip and onchip.get("kernels"):  # ncu pipe utilisation of the category's kernels, time weighted
        ks = list(onchip["kernels"].values())
        tw = sum(k_["us_ncu"] for k_ in ks) or 1.0
        roof["fp64_pipe_frac"] = sum(k_["us_ncu"] * k_["fp64_pipe_pct"] for k_ in ks) / tw / 100.0
        roof["l1_data_pipe_frac"] = sum(k_["us_ncu"] * k_["l1tex_pct"] for k_ in ks) / tw / 100.0
    out["roofline"] = roof
    out["kernel_time_ms_per_solve"] = {k_: v[0] for k_, v in table.items()}
    out["kernel_launches_per_solve"] = {k_: v[1] for k_, v in table.items()}

    # e2e: the public API with HOST buffers (pinned): the C-ABI's host path uploads b, solves, and
    # copies x back (overlapped with the true-residual check); wall clock around synchronous calls
    res = None
    del b, x, y
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    b_pin = torch.from_numpy(b_host).pin_memory()
    x_pin = torch.empty_like(b_pin).pin_memory()
    b_pin_np, x_pin_np = b_pin.numpy(), x_pin.numpy()
    with torch.cuda.stream(stream):
        fp.gmres_right(op, plan, b_pin_np, cfg, out=x_pin_np)
        if sync:
            sync()
        t0 = time.perf_counter()
        for _ in range(steps):
            r_e2e = fp.gmres_right(op, plan, b_pin_np, cfg, out=x_pin_np)
        t_e2e = (time.perf_counter() - t0) / steps
        stream.synchronize()
    out["e2e"] = {"value": 1.0 / t_e2e, "unit": UNIT, "h2d_bytes_per_step": 8 * N, "d2h_bytes_per_step": 8 * N,
                  "iterations": int(r_e2e.report.iterations),
                  "x_matches_device": bool(np.array_equal(x_pin_np[::1009], x_sample))}
    del op, plan, b_pin, x_pin
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2, help="headline BASELINE config (default 2)")
    ap.add_argument("--gamma", type=float, default=1.2, help="config 1 only")
    ap.add_argument("--secondary", default="1,3", help="BASELINE configs measured after the headline ('' = none)")
    ap.add_argument("--ref-steps", type=int, default=0,
                    help="reference arm: cap on the full solves timed (0 = --steps; FPC_REF_BUDGET_S bounds the run)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "p2p"],
                    help="N > 1 sharded solve: NCCL all_to_all exchanges, or peer-store kernels into "
                         "CUDA-IPC-shared receive buffers (kernels_p2p.cu)")
    ap.add_argument("--ordering", default="reference", choices=["reference", "commuted"],
                    help="PC factor ordering: reference (time FFT, tau solves, inverse FFT) or commuted (SURVEY 8(f)1)")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: independent replicas instead of the sharded solve")
    ap.add_argument("--sweep", action="store_true", help="BASELINE config 4: PC apply + matvec sweep (JSON per point)")
    ap.add_argument("--sweep-nx", default="", help="comma list (default 1023..65535)")
    ap.add_argument("--sweep-nt", default="", help="comma list (default 256..8192)")
    ap.add_argument("--sweep-reps", type=int, default=50)
    ap.add_argument("--sweep-sharded", action="store_true",
                    help="config 4 through the sharded (torchrun) path even at N = 1")
    ap.add_argument("--sweep-cpu-max", type=float, default=4e6, help="largest N timed on the CPU reference")
    args = ap.parse_args()
    if args.sweep:
        run_sweep(args)
        return
    args.steps_ref = max(1, min(args.steps, args.ref_steps) if args.ref_steps > 0 else args.steps)
    args.warmup_ref = max(0, args.warmup)

    from paper_2003_07020_b200 import problems
    w = problems.config(args.config, args.gamma if args.config == 1 else None)

    if args.impl == "reference":
        run_reference(args, w)
        return

    import torch
    import torch.distributed as dist
    rank, world, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 and not args.replicas:
        run_sharded(args, w, rank, world, local)
        return

    import paper_2003_07020_b200 as fp
    stream = torch.cuda.Stream(device=dev)
    ctx = fp.Context(local, stream)
    sync = dist.barrier if world > 1 else None

    def max_over_ranks(t):
        if world == 1:
            return t
        tt = torch.tensor([t], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    m = measure(fp, torch, w, args, stream, ctx, dev, args.steps, args.warmup, True, sync)
    t_step = max_over_ranks(m["ms_per_step"] * 1e-3)
    t_e2e = max_over_ranks(1.0 / m["e2e"]["value"])
    m["e2e"]["value"] = world / t_e2e

    # secondary BASELINE configs (same run, fewer steps; config 3 is 8.6 GB per Krylov vector)
    secondary = {}
    for c in [int(v) for v in args.secondary.split(",") if v.strip()]:
        if c == args.config:
            continue
        ws = problems.config(c, 1.2 if c == 1 else None)
        try:
            big = ws.dim > 2e8
            r = measure(fp, torch, ws, args, stream, ctx, dev, 2 if big else min(args.steps, 5),
                        1 if big else min(args.warmup, 3), False, sync)
            r["config"] = workload_config(ws)
            secondary[ws.name] = r
        except Exception as e:  # noqa: BLE001
            secondary[ws.name] = {"error": str(e)[:300]}
        torch.cuda.empty_cache()

    # CPU baseline: the reference on this host (rank 0, N = 1 only): ONE full solve of the headline
    # workload at all host threads (the reference's own report.seconds)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            threads = os.cpu_count() or 1
            sec, its = cpu_reference_solve(w, threads)
            cpu = {"value": 1.0 / sec, "unit": UNIT, "cores": threads, "kind": "reference",
                   "sample": f"one full reference gmres_right solve (oracle/_ref) of {w.name}, {its} iterations, "
                             f"{sec:.1f} s (report.seconds, krylov.hpp:87-190)", "cpu_model": cpu_model()}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        cfg = workload_config(w)
        cfg.update({"parallelism": f"replicas x{world}" if world > 1 else "single GPU", "pc_ordering": args.ordering,
                    "l2": f"inputs larger than L2 ({8 * w.dim / 1e6:.0f} MB per Krylov vector vs 126 MB L2)"})
        line = {
            "metric": METRIC, "value": world / t_step, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded uniform[-1,1] source, u0 = " + ("x^2(1-x)^2 y^2(1-y)^2)" if w.two_dim else "x^2(1-x)^2)"),
            "config": cfg, "time_to_tol_s": t_step,
        }
        for key in ("iterations", "restarts", "true_relative_residual", "pc_applies_per_s", "matvecs_per_s",
                    "pc_apply_gbs", "matvec_gbs", "e2e", "gpu_launches", "roofline", "solve_roofline",
                    "kernel_time_ms_per_solve", "kernel_launches_per_solve", "clocks"):
            line[key] = m.get(key)
        line["secondary"] = secondary
        line["cpu_baseline"] = cpu
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
