"""Sizes outside the power-of-two kernels (the reference's Bluestein fallback, fft.hpp:69-101): any
n_time <= 4096 and any DST length n_space <= 2047 run the PC apply on kernels_generic.cu (Bluestein
transforms on the device), the matvec on the regular kernels (its circulant embedding is always a
power of two, toeplitz.hpp:26).  Parity against the C oracle, which restates the reference's
Bluestein path."""
import numpy as np
import pytest

import paper_2003_07020_b200 as fp
from paper_2003_07020_b200 import problems

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


# (1.5, 777, 1200): 1200 rows of 777 points run the matvec on the one-warp-per-row kernels
# (kernels_warp32.cu) with a ragged zero-padded row; (.., 603, 3) in 2D: their column pass with a
# partial last tile (603 = 8 * 75 + 3)
CASES_1D = [(1.5, 100, 10), (1.3, 1000, 7), (1.7, 2047, 3), (1.5, 500, 64), (1.8, 255, 12), (1.2, 6, 5),
            (1.5, 777, 1200),
            (1.5, 5000, 16)]  # the last: Ns > 2047 with Nt a power of two -> NotImplementedError
CASES_2D = [(1.3, 1.7, 20, 6), (1.5, 1.5, 50, 16), (1.4, 1.2, 31, 12), (1.6, 1.3, 603, 3)]


def prob_1d(gamma, ns, nt):
    h, dt = 1.0 / (ns + 1), 1.0 / nt
    return fp.AllAtOnceOperator(fp.TimeStencil(nt), fp.RieszJacobian1D(gamma, 1.0, h, ns), dt), h, dt


@pytest.mark.parametrize("gamma,ns,nt", CASES_1D)
def test_generic_1d_operators(oracle, gamma, ns, nt):
    if ns > 2047:
        with pytest.raises(NotImplementedError):
            prob_1d(gamma, ns, nt)
        return
    op, h, dt = prob_1d(gamma, ns, nt)
    plan = fp.build_plan(fp.PreconditionerKind.generalized(), nt, dt, op)
    po = oracle.problem_1d(gamma, 1.0, h, ns, nt, dt).build_plan()
    # the tau spectrum's smallest eigenvalue is a cancellation (tau.hpp:46-53): the margin agrees to
    # the ulp-level differences of two Bluestein restatements amplified by it
    assert abs(plan.min_shift_margin - po.min_shift_margin) <= 1e-9 * po.min_shift_margin
    v = np.random.default_rng(ns + 31 * nt).uniform(-1, 1, ns * nt)
    assert rel(op.apply(v), po.matvec(v)) <= 1e-13
    # Bar 1e-10 (looser than the power-of-two path's 1e-12): the device's Bluestein transforms run
    # in radix-16 Stockham passes, the reference's in radix-2 (fft.hpp:49-89); the rounding
    # difference (~1e-15) is amplified by the alpha^{-k/Nt} scalings (up to 1/alpha = 2 Nt) and by
    # the smallest shifted eigenvalues lambda - dt sigma the tau solve divides by.
    from oracle import oracle as O
    assert O.Reference.available()
    pr = O.Reference().problem_1d(gamma, 1.0, h, ns, nt, dt).build_plan()
    z_gpu, z_orc, z_ref = fp.apply_inverse(plan, v), po.pc_apply(v), pr.pc_apply(v)
    assert rel(z_gpu, z_ref) <= 1e-10 and rel(z_gpu, z_orc) <= 1e-10
    zf = fp.apply_inverse(plan, v, sweep=fp.InnerSweep.full)
    assert rel(zf, z_gpu) <= 1e-11  # half and full sweeps agree (test_pint.cpp:203-216)
    assert rel(fp.apply_forward(plan, v), po.pc_forward(v)) <= 1e-9
    # forward after inverse is the identity (test_pint.cpp:188-201)
    assert rel(fp.apply_forward(plan, fp.apply_inverse(plan, v)), v) <= 1e-10


@pytest.mark.parametrize("gx,gy,n,nt", CASES_2D)
def test_generic_2d_operators(oracle, gx, gy, n, nt):
    h, dt = 1.0 / (n + 1), 1.0 / nt
    op = fp.AllAtOnceOperator(fp.TimeStencil(nt), fp.RieszJacobian2D(gx, gy, 1.0, 1.0, h, n), dt)
    plan = fp.build_plan(fp.PreconditionerKind.generalized(), nt, dt, op)
    po = oracle.problem_2d(gx, gy, 1.0, 1.0, h, n, nt, dt).build_plan()
    v = np.random.default_rng(n + 7 * nt).uniform(-1, 1, n * n * nt)
    assert rel(op.apply(v), po.matvec(v)) <= 1e-13
    assert rel(fp.apply_inverse(plan, v), po.pc_apply(v)) <= 1e-11
    assert rel(fp.apply_forward(plan, v), po.pc_forward(v)) <= 1e-11


@pytest.mark.parametrize("two_dim,n,nt,restart", [(False, 200, 24, 0), (False, 999, 100, 20), (True, 40, 10, 5)])
def test_generic_gmres(oracle, two_dim, n, nt, restart):
    if two_dim:
        w = problems.workload_2d(1.3, 1.7, n + 1, nt)
        op = fp.AllAtOnceOperator(fp.TimeStencil(nt), fp.RieszJacobian2D(1.3, 1.7, 1.0, 1.0, w.h, n), w.dt)
        po = oracle.problem_2d(1.3, 1.7, 1, 1, w.h, n, nt, w.dt).build_plan()
    else:
        w = problems.workload_1d(1.5, n + 1, nt)
        op = fp.AllAtOnceOperator(fp.TimeStencil(nt), fp.RieszJacobian1D(1.5, 1.0, w.h, n), w.dt)
        po = oracle.problem_1d(1.5, 1.0, w.h, n, nt, w.dt).build_plan()
    plan = fp.build_plan(fp.PreconditionerKind.generalized(), nt, w.dt, op)
    b = problems.rhs(w)
    res = fp.gmres_right(op, plan, b, fp.SolverConfig(tol=1e-10, max_iter=200, restart=restart))
    xo, ro = po.gmres(b, 1e-10, 200, restart=restart)
    assert res.report.converged and ro.converged
    assert abs(res.report.iterations - ro.iterations) <= 1
    assert rel(res.x, xo) <= 1e-10


def test_generic_rejects_commuted_and_sharding():
    op, h, dt = prob_1d(1.5, 100, 10)
    with pytest.raises(NotImplementedError):
        fp.build_plan(fp.PreconditionerKind.generalized(), 10, dt, op, ordering=fp.Ordering.commuted)
