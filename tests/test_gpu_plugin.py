"""The reference's plugin interface (krylov.hpp:83-85: gmres_right over any callables
void(span<const double>, span<double>)) in both directions, through the C-ABI:
  * the library's generic gmres_right over host callables (fpc_gmres_callbacks), and
  * the UNMODIFIED reference's own gmres_right (oracle/_ref) driving the library's fpc_matvec /
    fpc_pc_apply as its callables -- the integration a reference maintainer would write."""
import numpy as np
import pytest

import paper_2003_07020_b200 as fp
from paper_2003_07020_b200 import problems

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def setup(gamma=1.5, ns=255, nt=64, two_dim=False):
    if two_dim:
        w = problems.workload_2d(1.3, 1.7, ns + 1, nt)
        jac = fp.RieszJacobian2D(1.3, 1.7, 1.0, 1.0, w.h, w.n)
    else:
        w = problems.workload_1d(gamma, ns + 1, nt)
        jac = fp.RieszJacobian1D(gamma, 1.0, w.h, ns)
    op = fp.AllAtOnceOperator(fp.TimeStencil(nt), jac, w.dt)
    plan = fp.build_plan(fp.PreconditionerKind.generalized(), nt, w.dt, op)
    return w, op, plan, problems.rhs(w)


@pytest.mark.parametrize("restart,two_dim", [(0, False), (5, False), (0, True)])
def test_generic_gmres_over_host_callables(oracle, restart, two_dim):
    w, op, plan, b = setup(ns=31 if two_dim else 255, nt=16 if two_dim else 64, two_dim=two_dim)
    cfg = fp.SolverConfig(tol=1e-10, max_iter=200, restart=restart)
    calls = {"a": 0, "p": 0}

    def apply_a(v, out):
        calls["a"] += 1
        op.apply(v, out)

    def apply_pinv(v, out):
        calls["p"] += 1
        fp.apply_inverse(plan, v, out)

    g = fp.gmres_right_callables(op.dim(), apply_a, apply_pinv, b, cfg)
    d = fp.gmres_right(op, plan, b, cfg)
    po = (oracle.problem_2d(1.3, 1.7, 1, 1, w.h, w.n, w.n_time, w.dt) if two_dim
          else oracle.problem_1d(w.gamma[0], 1.0, w.h, w.n, w.n_time, w.dt)).build_plan()
    xo, ro = po.gmres(b, 1e-10, 200, restart=restart)
    assert g.report.converged and abs(g.report.iterations - ro.iterations) <= 1
    assert abs(g.report.iterations - d.report.iterations) <= 1
    assert rel(g.x, xo) <= 1e-10 and rel(g.x, d.x) <= 1e-10
    assert g.report.true_relative_residual <= 1e-9
    # one P^{-1} and one A per step, plus x = P^{-1} V y per cycle and the residuals
    k = int(g.report.iterations)
    assert calls["p"] == k + g.report.restarts + 1
    assert calls["a"] >= k + 1


def test_generic_gmres_callable_error_propagates():
    w, op, plan, b = setup(ns=63, nt=16)

    def bad(v, out):
        raise ArithmeticError("callable failed")

    with pytest.raises(ArithmeticError):
        fp.gmres_right_callables(op.dim(), bad, lambda v, o: fp.apply_inverse(plan, v, o), b)


@pytest.mark.parametrize("cfg_idx", [0, 2])
def test_reference_gmres_drives_b200_operators(cfg_idx):
    """The unmodified reference Krylov layer (krylov.hpp:83-192) with the B200 operators plugged in
    as its apply_a / apply_pinv -- against the reference's all-CPU solve on the same input.
    Config 0 at full size; config 2's parameters on a reduced 2D grid."""
    from oracle import oracle as O
    assert O.Reference.available(), "oracle/_ref missing (shipped prebuilt to the GPU box)"
    ref = O.Reference()
    if cfg_idx == 0:
        w = problems.config(0)
        jac = fp.RieszJacobian1D(w.gamma[0], 1.0, w.h, w.n)
        pr = ref.problem_1d(w.gamma[0], 1.0, w.h, w.n, w.n_time, w.dt).build_plan()
    else:
        w = problems.workload_2d(1.3, 1.7, 64, 64)
        jac = fp.RieszJacobian2D(1.3, 1.7, 1.0, 1.0, w.h, w.n)
        pr = ref.problem_2d(1.3, 1.7, 1.0, 1.0, w.h, w.n, w.n_time, w.dt).build_plan()
    op = fp.AllAtOnceOperator(fp.TimeStencil(w.n_time), jac, w.dt)
    plan = fp.build_plan(fp.PreconditionerKind.generalized(), w.n_time, w.dt, op)
    b = problems.rhs(w)
    x_mix, rep = ref.gmres_callables(op.dim(), lambda v, o: op.apply(v, o),
                                     lambda v, o: fp.apply_inverse(plan, v, o), b, w.tol, 200)
    x_ref, rr = pr.gmres(b, w.tol, 200)
    assert rep["converged"] and rr.converged
    assert rep["iterations"] == rr.iterations
    assert rel(x_mix, x_ref) <= 1e-10
    assert np.allclose(np.log10(rep["residual_history"]), np.log10(rr.residual_history), atol=0.05)
