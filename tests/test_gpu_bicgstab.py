"""BiCGSTAB (krylov.hpp:204-280) on the B200 vs the C oracle on seeded cases: 1D/2D, generalized
and Strang (alpha = 1) plans, half-step convergence, host and device buffers, zero rhs."""
import numpy as np
import pytest

import paper_2003_07020_b200 as fp
from paper_2003_07020_b200 import problems

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


CASES = [  # (dim, gammas, n, nt, alpha)
    (1, (1.5,), 255, 64, 0.0),
    (1, (1.2,), 1023, 128, 0.0),
    (1, (1.8,), 511, 32, 1.0),
    (2, (1.3, 1.7), 31, 32, 0.0),
    (2, (1.5, 1.5), 63, 16, 1.0),
]


@pytest.mark.parametrize("case", CASES)
def test_bicgstab_vs_oracle(oracle, case):
    dim, gm, n, nt, alpha = case
    h, dt = 1.0 / (n + 1), 1.0 / nt
    if dim == 1:
        jac = fp.RieszJacobian1D(gm[0], 1.0, h, n)
        po = oracle.problem_1d(gm[0], 1.0, h, n, nt, dt).build_plan(alpha)
        ns = n
    else:
        jac = fp.RieszJacobian2D(gm[0], gm[1], 1.0, 1.0, h, n)
        po = oracle.problem_2d(gm[0], gm[1], 1.0, 1.0, h, n, nt, dt).build_plan(alpha)
        ns = n * n
    op = fp.AllAtOnceOperator(fp.TimeStencil(nt), jac, dt)
    kind = fp.PreconditionerKind.generalized() if alpha <= 0 else fp.PreconditionerKind.with_alpha(alpha)
    plan = fp.build_plan(kind, nt, dt, op)
    b = np.random.default_rng(7 + n + nt).uniform(-1, 1, ns * nt)
    res = fp.bicgstab_left(op, plan, b, fp.SolverConfig(tol=1e-10, max_iter=200))
    xo, ro = po.bicgstab(b, 1e-10, 200)
    assert res.report.converged and ro.converged
    assert abs(res.report.iterations - ro.iterations) <= 1.0
    assert rel(res.x, xo) <= 1e-10
    assert len(res.report.residual_history) >= 1
    assert res.report.true_relative_residual <= 1e-9


def test_bicgstab_device_buffers_and_zero_rhs(oracle):
    import torch
    w = problems.workload_1d(1.5, 256, 64)
    op = fp.AllAtOnceOperator(fp.TimeStencil(w.n_time), fp.RieszJacobian1D(1.5, 1.0, w.h, w.n), w.dt)
    plan = fp.build_plan(fp.PreconditionerKind.generalized(), w.n_time, w.dt, op)
    b = problems.rhs(w)
    bd = torch.from_numpy(b).cuda()
    res = fp.bicgstab_left(op, plan, bd, fp.SolverConfig(tol=1e-10, max_iter=100))
    torch.cuda.synchronize()
    xh = fp.bicgstab_left(op, plan, b, fp.SolverConfig(tol=1e-10, max_iter=100))
    assert np.array_equal(res.x.cpu().numpy(), xh.x)  # deterministic reductions
    z = fp.bicgstab_left(op, plan, np.zeros_like(b))
    assert z.report.converged and z.report.iterations == 0 and not np.any(z.x)
    # half-step convergence counts k + 0.5 (krylov.hpp:244-249): a loose tolerance stops early
    r = fp.bicgstab_left(op, plan, b, fp.SolverConfig(tol=1.25, max_iter=100))  # first half step: 1.20
    assert r.report.converged and r.report.iterations == 0.5
