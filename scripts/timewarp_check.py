"""Parity of the warp-owned n_time = 1024 time FFTs (kernels_time_warp.cu) against the C oracle
(PC apply, forward action, full sweep) and against the split kernels (FPC_TIME_WARP=0 in a child).
Development aid."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2003_07020_b200 as fp
from oracle import oracle as O

rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
orc = O.Oracle()
nt = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
for (g, n) in [(1.5, 8191), (1.2, 4095), (1.8, 2371 * 2 + 1)]:
    if (n + 1) & n:
        continue
    h, dt = 1.0 / (n + 1), 1.0 / nt
    op = fp.AllAtOnceOperator(fp.TimeStencil(nt), fp.RieszJacobian1D(g, 1.0, h, n), dt)
    po = orc.problem_1d(g, 1.0, h, n, nt, dt)
    v = np.random.default_rng(n).uniform(-1, 1, n * nt)
    plan = fp.build_plan(fp.PreconditionerKind.generalized(), nt, dt, op)
    pp = po.build_plan()
    print("1D", n, nt, "pc", rel(fp.apply_inverse(plan, v), pp.pc_apply(v)), "fwd",
          rel(fp.apply_forward(plan, v), pp.pc_forward(v)), flush=True)
n = 127
h, dt = 1.0 / (n + 1), 1.0 / nt
op = fp.AllAtOnceOperator(fp.TimeStencil(nt), fp.RieszJacobian2D(1.3, 1.7, 1.0, 1.0, h, n), dt)
po = orc.problem_2d(1.3, 1.7, 1.0, 1.0, h, n, nt, dt)
v = np.random.default_rng(n).uniform(-1, 1, n * n * nt)
plan = fp.build_plan(fp.PreconditionerKind.generalized(), nt, dt, op)
pp = po.build_plan()
print("2D", n, nt, "pc", rel(fp.apply_inverse(plan, v), pp.pc_apply(v)), "fwd",
      rel(fp.apply_forward(plan, v), pp.pc_forward(v)), flush=True)
