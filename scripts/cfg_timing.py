"""Matvec / PC apply / solve times (device events) for BASELINE configs given on the command line
(e.g. 0 2); development A/B aid (FPC_LIB selects a variant build)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2003_07020_b200 as fp
from paper_2003_07020_b200 import problems

dev = torch.device("cuda", 0)
st = torch.cuda.Stream(device=dev)
ctx = fp.Context(0, st)
for c in [int(a) for a in sys.argv[1:]]:
    w = problems.config(c)
    jac = (fp.RieszJacobian2D(w.gamma[0], w.gamma[1], 1.0, 1.0, w.h, w.n) if w.two_dim
           else fp.RieszJacobian1D(w.gamma[0], 1.0, w.h, w.n))
    op = fp.AllAtOnceOperator(fp.TimeStencil(w.n_time), jac, w.dt, ctx)
    plan = fp.build_plan(fp.PreconditionerKind.generalized(), w.n_time, w.dt, op)
    b = torch.from_numpy(problems.rhs(w)).to(dev)
    y = torch.empty_like(b)
    cfg = fp.SolverConfig(tol=w.tol, max_iter=200, restart=w.restart)

    def t(fn, reps):
        for _ in range(2):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            fn()
        e1.record(st)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps
    tmv = t(lambda: op.apply(b, y), 10)
    tpc = t(lambda: fp.apply_inverse(plan, b, y), 10)
    tsol = t(lambda: fp.gmres_right(op, plan, b, cfg, out=y), 3)
    with fp.KernelProfile() as prof:
        r = fp.gmres_right(op, plan, b, cfg, out=y)
    print(f"cfg{c} matvec {tmv*1e3:.1f} us  pc {tpc*1e3:.1f} us  solve {tsol:.3f} ms  it {r.report.iterations}",
          {k: round(v[0] / v[1] * 1e3, 1) for k, v in prof.table.items()}, flush=True)
