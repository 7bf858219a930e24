"""PC apply / matvec device time with the per-kernel split at 1D n x n_time (development aid).
Usage: python scripts/pc_timing.py n n_time"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2003_07020_b200 as fp
n, nt = int(sys.argv[1]), int(sys.argv[2])
h, dt = 1.0 / (n + 1), 1.0 / nt
op = fp.AllAtOnceOperator(fp.TimeStencil(nt), fp.RieszJacobian1D(1.5, 1.0, h, n), dt)
plan = fp.build_plan(fp.PreconditionerKind.generalized(), nt, dt, op)
b = torch.randn(n * nt, dtype=torch.float64, device="cuda")
y = torch.empty_like(b)
for name, fn in (("matvec", lambda: op.apply(b, y)), ("pc", lambda: fp.apply_inverse(plan, b, y))):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): fn()
    e1.record(); torch.cuda.synchronize()
    with fp.KernelProfile() as prof:
        fn()
    print(n, nt, name, f"{e0.elapsed_time(e1) / 10:.3f} ms", {k: round(v[0] / v[1], 3) for k, v in prof.table.items()})
