"""1D n = 1023 x n_time: matvec / PC apply device time per (n_time), for the row-count threshold of the
one-warp-per-row kernels (FPC_W32_MIN_ROWS, FPC_W32).  Development aid."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2003_07020_b200 as fp
n = 1023
out = []
for nt in (256, 512, 1024, 2048, 4096, 8192):
    h, dt = 1.0 / (n + 1), 1.0 / nt
    op = fp.AllAtOnceOperator(fp.TimeStencil(nt), fp.RieszJacobian1D(1.5, 1.0, h, n), dt)
    plan = fp.build_plan(fp.PreconditionerKind.generalized(), nt, dt, op)
    b = torch.randn(n * nt, dtype=torch.float64, device="cuda")
    y = torch.empty_like(b)
    r = [nt]
    for fn in (lambda: op.apply(b, y), lambda: fp.apply_inverse(plan, b, y)):
        for _ in range(5): fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50): fn()
        e1.record(); torch.cuda.synchronize()
        r.append(round(e0.elapsed_time(e1) / 50 * 1e3, 1))
    out.append(tuple(r))
print("nt, matvec us, pc us:", out)
