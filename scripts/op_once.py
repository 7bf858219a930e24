"""One matvec and one PC apply of a BASELINE config (for ncu captures of the 2D kernels)."""
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
b = torch.from_numpy(problems.rhs(w)).cuda()
y = torch.empty_like(b)
op.apply(b, y)
fp.apply_inverse(plan, b, y)
torch.cuda.synchronize()
if len(sys.argv) > 2 and sys.argv[2] == "commuted":
    planc = fp.build_plan(fp.PreconditionerKind.generalized(), w.n_time, w.dt, op, ordering=fp.Ordering.commuted)
    fp.apply_inverse(planc, b, y)
    torch.cuda.synchronize()
