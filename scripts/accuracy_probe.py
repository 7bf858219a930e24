"""Accuracy probe: GPU vs C oracle vs the reference (oracle/_ref) on one workload."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2003_07020_b200 as fp
from paper_2003_07020_b200 import problems
from oracle.oracle import Oracle, Reference

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 0
w = problems.config(idx, float(sys.argv[2]) if len(sys.argv) > 2 else None)
o, r = Oracle(), Reference()
if w.two_dim:
    jac = fp.RieszJacobian2D(w.gamma[0], w.gamma[1], 1.0, 1.0, w.h, w.n)
    po = o.problem_2d(w.gamma[0], w.gamma[1], 1, 1, w.h, w.n, w.n_time, w.dt).build_plan()
    pr = r.problem_2d(w.gamma[0], w.gamma[1], 1, 1, w.h, w.n, w.n_time, w.dt).build_plan()
else:
    jac = fp.RieszJacobian1D(w.gamma[0], 1.0, w.h, w.n)
    po = o.problem_1d(w.gamma[0], 1.0, w.h, w.n, w.n_time, w.dt).build_plan()
    pr = r.problem_1d(w.gamma[0], 1.0, w.h, w.n, w.n_time, w.dt).build_plan()
op = fp.AllAtOnceOperator(fp.TimeStencil(w.n_time), jac, w.dt)
plan = fp.build_plan(fp.PreconditionerKind.generalized(), w.n_time, w.dt, op)
rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
b = problems.rhs(w)
v = np.random.default_rng(1).uniform(-1, 1, w.dim)
print("matvec  gpu-ref %.2e  orc-ref %.2e" % (rel(op.apply(v), pr.matvec(v)), rel(po.matvec(v), pr.matvec(v))))
print("pc      gpu-ref %.2e  orc-ref %.2e" % (rel(fp.apply_inverse(plan, v), pr.pc_apply(v)), rel(po.pc_apply(v), pr.pc_apply(v))))
xr, rr = pr.gmres(b, w.tol, 200)
res = fp.gmres_right(op, plan, b, fp.SolverConfig(tol=w.tol, max_iter=200, restart=0))
xo, ro = po.gmres(b, w.tol, 200)
print("x       gpu-ref %.2e  orc-ref %.2e   iters gpu %d orc %d ref %d" % (rel(res.x, xr), rel(xo, xr), res.report.iterations, ro.iterations, rr.iterations))
print("TRR     gpu %.2e  orc %.2e  ref %.2e ; TRR of gpu x via ref matvec %.2e" % (res.report.true_relative_residual, ro.true_relative_residual, rr.true_relative_residual, np.linalg.norm(b - pr.matvec(res.x)) / np.linalg.norm(b)))
print("Ax on ref x: gpu-ref %.2e" % (rel(op.apply(xr), pr.matvec(xr))))
print("history gpu", ["%.2e" % h for h in res.report.residual_history[-3:]], "ref", ["%.2e" % h for h in rr.residual_history[-3:]])
