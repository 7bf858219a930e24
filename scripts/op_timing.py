"""Matvec and PC apply device times (+ per-kernel live times) of a BASELINE config, development aid."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2003_07020_b200 as fp
from paper_2003_07020_b200 import problems
w = problems.config(int(sys.argv[1]))
jac = (fp.RieszJacobian2D(w.gamma[0], w.gamma[1], 1.0, 1.0, w.h, w.n) if w.two_dim
       else fp.RieszJacobian1D(w.gamma[0], 1.0, w.h, w.n))
op = fp.AllAtOnceOperator(fp.TimeStencil(w.n_time), jac, w.dt)
plan = fp.build_plan(fp.PreconditionerKind.generalized(), w.n_time, w.dt, op)
b = torch.randn(w.dim, dtype=torch.float64, device="cuda")
y = torch.empty_like(b)
for name, fn in (("matvec", lambda: op.apply(b, y)), ("pc", lambda: fp.apply_inverse(plan, b, y))):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): fn()
    e1.record(); torch.cuda.synchronize()
    with fp.KernelProfile() as prof:
        fn()
    print(name, f"{e0.elapsed_time(e1) / 3:.3f} ms", {k: round(v[0] / v[1], 3) for k, v in prof.table.items()})
