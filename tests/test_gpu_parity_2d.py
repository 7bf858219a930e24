"""GPU parity of the 2D hot path (RieszJacobian2D, 2D tau solves) against the C oracle."""
import numpy as np
import pytest

import paper_2003_07020_b200 as fp
from paper_2003_07020_b200 import problems

pytestmark = pytest.mark.gpu

SIZES = [(1.4, 1.8, 3, 4), (1.3, 1.7, 7, 8), (1.5, 1.5, 15, 16), (1.3, 1.7, 31, 8), (1.9, 1.2, 63, 4),
         (1.3, 1.7, 127, 8), (1.3, 1.7, 255, 8), (1.5, 1.5, 511, 4), (1.5, 1.5, 1023, 4),
         (1.4, 1.6, 2047, 4)]


def make(gx, gy, n, nt, kx=1.0, ky=1.0):
    h = 1.0 / (n + 1)
    dt = 1.0 / nt
    op = fp.AllAtOnceOperator(fp.TimeStencil(nt), fp.RieszJacobian2D(gx, gy, kx, ky, h, n), dt)
    return op, h, dt


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("gx,gy,n,nt", SIZES)
def test_matvec_2d(oracle, gx, gy, n, nt):
    op, h, dt = make(gx, gy, n, nt)
    po = oracle.problem_2d(gx, gy, 1.0, 1.0, h, n, nt, dt)
    v = np.random.default_rng(n + nt).uniform(-1, 1, n * n * nt)
    assert rel(op.apply(v), po.matvec(v)) <= 1e-13


@pytest.mark.parametrize("gx,gy,n,nt", SIZES)
def test_pc_apply_2d(oracle, gx, gy, n, nt):
    op, h, dt = make(gx, gy, n, nt)
    plan = fp.build_plan(fp.PreconditionerKind.generalized(), nt, dt, op)
    po = oracle.problem_2d(gx, gy, 1.0, 1.0, h, n, nt, dt).build_plan()
    assert abs(plan.min_shift_margin - po.min_shift_margin) <= 1e-12 * po.min_shift_margin
    assert np.abs(op.tau_sigma() - po.sigma()).max() <= 1e-12 * np.abs(po.sigma()).max()
    v = np.random.default_rng(3 * n + nt).uniform(-1, 1, n * n * nt)
    assert rel(fp.apply_inverse(plan, v), po.pc_apply(v)) <= 1e-12


def test_pc_apply_2d_anisotropic(oracle):
    # distinct kappa_x, kappa_y and alpha (test_pint.cpp:173-186 uses (1.4,1.8,0.03,0.05,h=0.25))
    n, nt, dt = 7, 8, 0.2
    op = fp.AllAtOnceOperator(fp.TimeStencil(nt), fp.RieszJacobian2D(1.4, 1.8, 0.03, 0.05, 0.25, n), dt)
    plan = fp.build_plan(fp.PreconditionerKind.with_alpha(0.6), nt, dt, op)
    po = oracle.problem_2d(1.4, 1.8, 0.03, 0.05, 0.25, n, nt, dt).build_plan(0.6)
    v = np.random.default_rng(1).uniform(-1, 1, n * n * nt)
    assert rel(fp.apply_inverse(plan, v), po.pc_apply(v)) <= 1e-12
    assert rel(op.apply(v), po.matvec(v)) <= 1e-13


@pytest.mark.parametrize("gx,gy,n,nt,restart", [(1.3, 1.7, 31, 16, 0), (1.3, 1.7, 63, 32, 20),
                                                (1.5, 1.5, 127, 16, 10)])
def test_gmres_2d(oracle, gx, gy, n, nt, restart):
    w = problems.workload_2d(gx, gy, n + 1, nt)
    op = fp.AllAtOnceOperator(fp.TimeStencil(nt), fp.RieszJacobian2D(gx, gy, 1.0, 1.0, w.h, n), w.dt)
    plan = fp.build_plan(fp.PreconditionerKind.generalized(), nt, w.dt, op)
    b = problems.rhs(w)
    res = fp.gmres_right(op, plan, b, fp.SolverConfig(tol=1e-10, max_iter=200, restart=restart))
    po = oracle.problem_2d(gx, gy, 1.0, 1.0, w.h, n, nt, w.dt).build_plan()
    xo, ro = po.gmres(b, 1e-10, 200, restart=restart)
    assert res.report.converged and ro.converged
    assert abs(res.report.iterations - ro.iterations) <= 1
    assert rel(res.x, xo) <= 1e-10


def test_pc_forward_2d(oracle):
    n, nt, dt = 15, 8, 0.2
    op = fp.AllAtOnceOperator(fp.TimeStencil(nt), fp.RieszJacobian2D(1.4, 1.8, 0.03, 0.05, 0.25, n), dt)
    plan = fp.build_plan(fp.PreconditionerKind.with_alpha(0.6), nt, dt, op)
    po = oracle.problem_2d(1.4, 1.8, 0.03, 0.05, 0.25, n, nt, dt).build_plan(0.6)
    v = np.random.default_rng(2).uniform(-1, 1, n * n * nt)
    pv = fp.apply_forward(plan, v)
    assert rel(pv, po.pc_forward(v)) <= 1e-12
    assert rel(fp.apply_inverse(plan, pv), v) <= 1e-10


def test_full_sweep_2d(oracle):
    n, nt, dt = 15, 8, 0.125
    op = fp.AllAtOnceOperator(fp.TimeStencil(nt), fp.RieszJacobian2D(1.3, 1.7, 1.0, 1.0, 1 / 16, n), dt)
    plan = fp.build_plan(fp.PreconditionerKind.generalized(), nt, dt, op)
    po = oracle.problem_2d(1.3, 1.7, 1.0, 1.0, 1 / 16, n, nt, dt).build_plan()
    v = np.random.default_rng(4).uniform(-1, 1, n * n * nt)
    assert rel(fp.apply_inverse(plan, v, sweep=fp.InnerSweep.full), po.pc_apply(v, True)) <= 1e-12
