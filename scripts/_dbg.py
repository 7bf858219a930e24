import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2003_07020_b200 as fp
n, nt = 8191, 512
h, dt = 1.0/(n+1), 1.0/nt
op = fp.AllAtOnceOperator(fp.TimeStencil(nt), fp.RieszJacobian1D(1.5, 1.0, h, n), dt)
plan = fp.build_plan(fp.PreconditionerKind.generalized(), nt, dt, op)
b = torch.rand(nt*n, dtype=torch.float64, device="cuda")
y = torch.empty_like(b)
fp.apply_inverse(plan, b, y)
torch.cuda.synchronize()
print("ok", float(y.norm()))
