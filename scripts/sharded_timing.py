"""Sharded-solver overhead probe: ShardedSolver at world size 1 (no collectives) vs the fused
single-GPU solve, config 1 (development aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2003_07020_b200 as fp
from paper_2003_07020_b200 import problems
from paper_2003_07020_b200.distributed import CudaShardKernels, ShardedSolver
w = problems.config(1)
dev = torch.device("cuda", 0)
ctx = fp.Context(0, torch.cuda.current_stream(dev))
op = fp.AllAtOnceOperator(fp.TimeStencil(w.n_time), fp.RieszJacobian1D(w.gamma[0], 1.0, w.h, w.n), w.dt, ctx)
plan = fp.build_plan(fp.PreconditionerKind.generalized(), w.n_time, w.dt, op)
s = ShardedSolver(w.n_time, w.n_space, CudaShardKernels(op, plan))
b = torch.from_numpy(problems.rhs(w)).to(dev)
for _ in range(2):
    x, rep = s.gmres(b, w.tol, 200, w.restart)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3):
    x, rep = s.gmres(b, w.tol, 200, w.restart)
torch.cuda.synchronize()
t = (time.perf_counter() - t0) / 3
cfg = fp.SolverConfig(tol=w.tol, max_iter=200, restart=w.restart)
res = fp.gmres_right(op, plan, b, cfg)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3):
    res = fp.gmres_right(op, plan, b, cfg)
torch.cuda.synchronize()
t1 = (time.perf_counter() - t0) / 3
print(f"sharded G=1: {t*1e3:.2f} ms, {rep.iterations} it, TRR {rep.true_relative_residual:.3e}; fused: {t1*1e3:.2f} ms")
with fp.KernelProfile() as pr:
    s.gmres(b, w.tol, 200, w.restart)
print({k: (round(v[0], 2), v[1]) for k, v in pr.table.items()})
