"""Child process of tests/test_gpu_variants.py: the library's kernel-selection knobs are read from
the environment once per process, so every variant runs in its own interpreter.
usage: python tests/variant_child.py <out.npz> <case> ...   case = pc:<1d|2d>:<n>:<nt> | solve:<1d|2d>:<n>:<nt>"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2003_07020_b200 as fp  # noqa: E402

out = {}
for case in sys.argv[2:]:
    what, kind, n, nt = case.split(":")
    n, nt = int(n), int(nt)
    h, dt = 1.0 / (n + 1), 1.0 / nt
    jac = fp.RieszJacobian2D(1.3, 1.7, 1.0, 1.0, h, n) if kind == "2d" else fp.RieszJacobian1D(1.5, 1.0, h, n)
    op = fp.AllAtOnceOperator(fp.TimeStencil(nt), jac, dt)
    plan = fp.build_plan(fp.PreconditionerKind.generalized(), nt, dt, op)
    ns = n * n if kind == "2d" else n
    b = np.random.default_rng(11).uniform(-1.0, 1.0, nt * ns)
    if what == "pc":
        y = np.empty_like(b)
        fp.apply_inverse(plan, b, y)
        out[case] = y
        y2 = np.empty_like(b)
        op.apply(b, y2)
        out[case + ":mv"] = y2
    else:
        r = fp.gmres_right(op, plan, b, fp.SolverConfig(tol=1e-10, max_iter=200, restart=20))
        out[case] = r.x
        out[case + ":it"] = np.array([r.report.iterations, r.report.true_relative_residual])
np.savez(sys.argv[1], **out)
