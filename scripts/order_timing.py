"""Config-1 PC apply + GMRES solve time, reference vs commuted ordering (device events)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2003_07020_b200 as fp
from paper_2003_07020_b200 import problems

w = problems.config(1, 1.2)
dev = torch.device("cuda", 0)
st = torch.cuda.Stream(device=dev)
ctx = fp.Context(0, st)
op = fp.AllAtOnceOperator(fp.TimeStencil(w.n_time), fp.RieszJacobian1D(w.gamma[0], 1.0, w.h, w.n), w.dt, ctx)
b = torch.from_numpy(problems.rhs(w)).to(dev)
y = torch.empty_like(b)
cfg = fp.SolverConfig(tol=w.tol, max_iter=200, restart=w.restart)
for order in (fp.Ordering.reference, fp.Ordering.commuted):
    plan = fp.build_plan(fp.PreconditionerKind.generalized(), w.n_time, w.dt, op, ordering=order)
    def t(fn, reps):
        for _ in range(3): fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps): fn()
        e1.record(st); torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps
    tpc = t(lambda: fp.apply_inverse(plan, b, y), 20)
    tsolve = t(lambda: fp.gmres_right(op, plan, b, cfg, out=y), 5)
    with fp.KernelProfile() as prof:
        r = fp.gmres_right(op, plan, b, cfg, out=y)
    print(order.name, f"pc {tpc*1e3:.1f} us  solve {tsolve:.3f} ms  it {r.report.iterations} trr {r.report.true_relative_residual:.3e}",
          {k: round(v[0] / v[1] * 1e3, 1) for k, v in prof.table.items()})
