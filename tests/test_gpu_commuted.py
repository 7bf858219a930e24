"""Commuted preconditioner ordering on the B200 (kernels_commuted.cu) vs the C
oracle's reference-ordering apply: same operator up to rounding.  PC apply / forward at sizes across
every kernel instantiation (1D up to n_space = 65535, and 2D), GMRES iteration counts and x."""
import numpy as np
import pytest

import paper_2003_07020_b200 as fp
from paper_2003_07020_b200 import problems

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def make(gamma, ns, nt, alpha=0.0):
    h, dt = 1.0 / (ns + 1), 1.0 / nt
    op = fp.AllAtOnceOperator(fp.TimeStencil(nt), fp.RieszJacobian1D(gamma, 1.0, h, ns), dt)
    kind = fp.PreconditionerKind.generalized() if alpha <= 0 else fp.PreconditionerKind.with_alpha(alpha)
    return op, fp.build_plan(kind, nt, dt, op, ordering=fp.Ordering.commuted), h, dt


@pytest.mark.parametrize("ns,nt", [(3, 4), (15, 8), (31, 64), (255, 16), (1023, 256), (4095, 32),
                                   (8191, 64), (511, 2048), (127, 1024), (255, 2048), (127, 4096), (63, 8192),
                                   (63, 16384), (16383, 8), (32767, 4), (65535, 4)])
def test_commuted_pc_vs_oracle(oracle, ns, nt):
    op, plan, h, dt = make(1.5, ns, nt)
    po = oracle.problem_1d(1.5, 1.0, h, ns, nt, dt).build_plan()
    v = np.random.default_rng(ns * 7 + nt).uniform(-1, 1, ns * nt)
    assert rel(fp.apply_inverse(plan, v), po.pc_apply(v)) <= 1e-12
    assert rel(fp.apply_forward(plan, v), po.pc_forward(v)) <= 1e-12


@pytest.mark.parametrize("gamma,alpha", [(1.2, 0.0), (1.8, 1.0)])
def test_commuted_gmres_vs_oracle(oracle, gamma, alpha):
    ns, nt = 1023, 128
    op, plan, h, dt = make(gamma, ns, nt, alpha)
    po = oracle.problem_1d(gamma, 1.0, h, ns, nt, dt).build_plan(alpha)
    b = np.random.default_rng(3).uniform(-1, 1, ns * nt)
    res = fp.gmres_right(op, plan, b, fp.SolverConfig(tol=1e-10, max_iter=200, restart=20))
    xo, ro = po.gmres(b, 1e-10, 200, restart=20)
    assert abs(res.report.iterations - ro.iterations) <= 1
    assert rel(res.x, xo) <= 1e-10
    bi = fp.bicgstab_left(op, plan, b, fp.SolverConfig(tol=1e-10, max_iter=200))
    xb, rb = po.bicgstab(b, 1e-10, 200)
    assert abs(bi.report.iterations - rb.iterations) <= 1 and rel(bi.x, xb) <= 1e-10


def test_commuted_switch_and_rejections():
    op, plan, h, dt = make(1.5, 255, 64)
    v = np.random.default_rng(1).uniform(-1, 1, 255 * 64)
    zc = fp.apply_inverse(plan, v)
    plan.set_ordering(fp.Ordering.reference)
    zr = fp.apply_inverse(plan, v)
    assert rel(zc, zr) <= 1e-12
    op2 = fp.AllAtOnceOperator(fp.TimeStencil(10), fp.RieszJacobian1D(1.5, 1.0, 1 / 101, 100), 1 / 10)
    with pytest.raises(NotImplementedError):  # the Bluestein sizes run the reference ordering only
        fp.build_plan(fp.PreconditionerKind.generalized(), 10, 1 / 10, op2, ordering=fp.Ordering.commuted)
    with pytest.raises(ValueError):
        plan.set_ordering(7)


def make_2d(gx, gy, n, nt):
    h, dt = 1.0 / (n + 1), 1.0 / nt
    op = fp.AllAtOnceOperator(fp.TimeStencil(nt), fp.RieszJacobian2D(gx, gy, 1.0, 1.0, h, n), dt)
    return op, fp.build_plan(fp.PreconditionerKind.generalized(), nt, dt, op, ordering=fp.Ordering.commuted), h, dt


@pytest.mark.parametrize("gx,gy,n,nt", [(1.3, 1.7, 7, 8), (1.5, 1.5, 31, 16), (1.3, 1.7, 255, 32), (1.5, 1.2, 63, 1024),
                                        (1.5, 1.5, 1023, 4)])
def test_commuted_2d_pc_vs_oracle(oracle, gx, gy, n, nt):
    """2D commuted ordering: the 2D DST-I of every time level (rows then columns, tau.hpp:79-96),
    the per-mode time solve over the n^2 spatial modes, the 2D DST again."""
    op, plan, h, dt = make_2d(gx, gy, n, nt)
    po = oracle.problem_2d(gx, gy, 1.0, 1.0, h, n, nt, dt).build_plan()
    v = np.random.default_rng(n * 3 + nt).uniform(-1, 1, n * n * nt)
    assert rel(fp.apply_inverse(plan, v), po.pc_apply(v)) <= 1e-12
    assert rel(fp.apply_forward(plan, v), po.pc_forward(v)) <= 1e-12


def test_commuted_2d_gmres_config3_parameters(oracle):
    w = problems.workload_2d(1.5, 1.5, 64, 64, tol=1e-9, restart=10)
    op, plan, h, dt = make_2d(1.5, 1.5, w.n, w.n_time)
    b = problems.rhs(w)
    res = fp.gmres_right(op, plan, b, fp.SolverConfig(tol=w.tol, max_iter=200, restart=10))
    po = oracle.problem_2d(1.5, 1.5, 1, 1, w.h, w.n, w.n_time, w.dt).build_plan()
    xo, ro = po.gmres(b, w.tol, 200, restart=10)
    assert abs(res.report.iterations - ro.iterations) <= 1 and rel(res.x, xo) <= 1e-10
