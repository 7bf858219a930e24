"""Matvec and PC apply device times (+ per-kernel live times) at 2D n = 1023 x n_time (default 64):
the config-3 lattice kernels on a grid that still runs tens of waves.  Development aid.
Usage: python scripts/w32_timing.py [n_time] [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2003_07020_b200 as fp
nt = int(sys.argv[1]) if len(sys.argv) > 1 else 64
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
n = 1023
h, dt = 1.0 / (n + 1), 1.0 / nt
op = fp.AllAtOnceOperator(fp.TimeStencil(nt), fp.RieszJacobian2D(1.5, 1.5, 1.0, 1.0, h, n), dt)
plan = fp.build_plan(fp.PreconditionerKind.generalized(), nt, dt, op)
b = torch.randn(n * n * nt, dtype=torch.float64, device="cuda")
y = torch.empty_like(b)
for name, fn in (("matvec", lambda: op.apply(b, y)), ("pc", lambda: fp.apply_inverse(plan, b, y))):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    with fp.KernelProfile() as prof:
        fn()
    print(name, f"{e0.elapsed_time(e1) / reps:.3f} ms", {k: round(v[0] / v[1], 3) for k, v in prof.table.items()})
