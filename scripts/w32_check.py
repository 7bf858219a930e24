"""Parity of the n = 1023 warp-owned 1024-point kernels (kernels_warp32.cu) against the C oracle:
2D matvec / PC apply / forward at n = 1023, 1D matvec / PC apply at 1023 x 4096.  Development aid."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2003_07020_b200 as fp
from oracle import oracle as O

rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
orc = O.Oracle()
for (gx, gy, n, nt) in [(1.5, 1.5, 1023, 4), (1.3, 1.7, 1023, 6)]:
    h, dt = 1.0 / (n + 1), 1.0 / nt
    op = fp.AllAtOnceOperator(fp.TimeStencil(nt), fp.RieszJacobian2D(gx, gy, 1.0, 1.0, h, n), dt)
    po = orc.problem_2d(gx, gy, 1.0, 1.0, h, n, nt, dt)
    v = np.random.default_rng(n + nt).uniform(-1, 1, n * n * nt)
    print("2D", n, nt, "matvec", rel(op.apply(v), po.matvec(v)), flush=True)
    try:
        plan = fp.build_plan(fp.PreconditionerKind.generalized(), nt, dt, op)
        pp = po.build_plan()
        print("2D", n, nt, "pc", rel(fp.apply_inverse(plan, v), pp.pc_apply(v)),
              "fwd", rel(fp.apply_forward(plan, v), pp.pc_forward(v)), flush=True)
    except NotImplementedError as e:
        print("skip pc", e)
for (g, n, nt) in [(1.5, 1023, 4096)]:
    h, dt = 1.0 / (n + 1), 1.0 / nt
    op = fp.AllAtOnceOperator(fp.TimeStencil(nt), fp.RieszJacobian1D(g, 1.0, h, n), dt)
    po = orc.problem_1d(g, 1.0, h, n, nt, dt)
    v = np.random.default_rng(7).uniform(-1, 1, n * nt)
    plan = fp.build_plan(fp.PreconditionerKind.generalized(), nt, dt, op)
    pp = po.build_plan()
    print("1D", n, nt, "matvec", rel(op.apply(v), po.matvec(v)), "pc", rel(fp.apply_inverse(plan, v), pp.pc_apply(v)),
          "fwd", rel(fp.apply_forward(plan, v), pp.pc_forward(v)), flush=True)
