"""Quick device timings of the hot-path pieces (development aid; bench.py is the contract)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2003_07020_b200 as fp
from paper_2003_07020_b200 import problems

def timeit(fn, stream, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    for _ in range(reps): fn()
    e.record(stream)
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e-3

cfgs = [(0, None), (1, 1.2)] if len(sys.argv) < 2 else [(int(sys.argv[1]), None)]
for idx, g in cfgs:
    w = problems.config(idx, g)
    stream = torch.cuda.Stream()
    ctx = fp.Context(0, stream)
    op = fp.AllAtOnceOperator(fp.TimeStencil(w.n_time), fp.RieszJacobian1D(w.gamma[0], 1.0, w.h, w.n), w.dt, ctx)
    plan = fp.build_plan(fp.PreconditionerKind.generalized(), w.n_time, w.dt, op)
    N = w.dim
    b = torch.from_numpy(problems.rhs(w)).cuda()
    y = torch.empty_like(b)
    with torch.cuda.stream(stream):
        tm = timeit(lambda: op.apply(b, y), stream)
        tp = timeit(lambda: fp.apply_inverse(plan, b, y), stream)
    torch.cuda.synchronize()
    t0 = time.time()
    res = fp.gmres_right(op, plan, b, fp.SolverConfig(tol=w.tol, max_iter=200, restart=w.restart))
    t1 = time.time()
    res = fp.gmres_right(op, plan, b, fp.SolverConfig(tol=w.tol, max_iter=200, restart=w.restart))
    t2 = time.time()
    print(f"{w.name}: N={N} matvec {tm*1e6:.1f} us ({16*N/tm/1e9:.0f} GB/s alg)  "
          f"pc {tp*1e6:.1f} us ({(16*N+64*(w.n_time//2+1)*w.n_space)/tp/1e9:.0f} GB/s alg)  "
          f"gmres iters {res.report.iterations} TRR {res.report.true_relative_residual:.2e} "
          f"solve {res.report.seconds*1e3:.2f} ms (first {1e3*(t1-t0):.1f} ms)")
