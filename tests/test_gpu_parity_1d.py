"""GPU parity of the 1D hot path against the C oracle (oracle/fracpint_oracle.c, itself pinned to
the reference in test_oracle_pins.py).  All calls go through the C-ABI (libfracpint_b200.so)."""
import numpy as np
import pytest

import paper_2003_07020_b200 as fp
from paper_2003_07020_b200 import problems

pytestmark = pytest.mark.gpu

# (gamma, n_space, n_time): every size class of the smem FFT engine for the Toeplitz (L = 2(n+1)),
# the DST (M = n+1) and the time FFT (Nt)
SIZES = [(1.5, 3, 4), (1.5, 7, 8), (1.3, 15, 16), (1.8, 31, 8), (1.5, 63, 32), (1.2, 127, 64),
         (1.7, 255, 128), (1.5, 511, 16), (1.5, 1023, 256), (1.9, 2047, 32), (1.4, 4095, 16),
         (1.2, 8191, 8), (1.5, 16383, 4), (1.3, 32767, 4), (1.7, 65535, 4)]


def make(gamma, ns, nt, kappa=1.0):
    h = 1.0 / (ns + 1)
    dt = 1.0 / nt
    st = fp.TimeStencil(nt)
    op = fp.AllAtOnceOperator(st, fp.RieszJacobian1D(gamma, kappa, h, ns), dt)
    return op, h, dt


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("gamma,ns,nt", SIZES)
def test_matvec_1d(oracle, gamma, ns, nt):
    op, h, dt = make(gamma, ns, nt)
    po = oracle.problem_1d(gamma, 1.0, h, ns, nt, dt)
    v = np.random.default_rng(ns * 7 + nt).uniform(-1, 1, ns * nt)
    y = op.apply(v)
    assert rel(y, po.matvec(v)) <= 1e-13


@pytest.mark.parametrize("gamma,ns,nt", SIZES)
def test_pc_apply_1d(oracle, gamma, ns, nt):
    op, h, dt = make(gamma, ns, nt)
    plan = fp.build_plan(fp.PreconditionerKind.generalized(), nt, dt, op)
    po = oracle.problem_1d(gamma, 1.0, h, ns, nt, dt).build_plan()
    assert abs(plan.alpha - po.alpha) == 0.0
    assert abs(plan.min_shift_margin - po.min_shift_margin) <= 1e-12 * po.min_shift_margin
    v = np.random.default_rng(ns * 11 + nt).uniform(-1, 1, ns * nt)
    z = fp.apply_inverse(plan, v)
    assert rel(z, po.pc_apply(v)) <= 1e-12


@pytest.mark.parametrize("gamma,ns,nt", [(1.5, 63, 512), (1.7, 255, 1024), (1.3, 31, 2048), (1.5, 127, 4096),
                                         (1.5, 15, 8192), (1.2, 1023, 2048), (1.4, 8191, 512)])
def test_pc_apply_long_time(oracle, gamma, ns, nt):
    # Nt = 1024 / 2048 run the parity-split 2-CTA time FFT kernels (kernels_tsplit.cu), Nt = 4096 /
    # 8192 the 4/8-CTA ones (kernels_tsplitc.cu), the other lengths the 1-CTA column kernels; ragged last tiles (Ns not a multiple of the tile width) included
    op, h, dt = make(gamma, ns, nt)
    plan = fp.build_plan(fp.PreconditionerKind.generalized(), nt, dt, op)
    po = oracle.problem_1d(gamma, 1.0, h, ns, nt, dt).build_plan()
    v = np.random.default_rng(ns * 13 + nt).uniform(-1, 1, ns * nt)
    assert rel(fp.apply_inverse(plan, v), po.pc_apply(v)) <= 1e-12
    assert rel(fp.apply_forward(plan, v), po.pc_forward(v)) <= 1e-12


@pytest.mark.parametrize("alpha", [0.5, 1e-3, 1.0])
def test_pc_apply_alpha(oracle, alpha):
    op, h, dt = make(1.5, 63, 16)
    plan = fp.build_plan(fp.PreconditionerKind.with_alpha(alpha), 16, dt, op)
    po = oracle.problem_1d(1.5, 1.0, h, 63, 16, dt).build_plan(alpha)
    v = np.random.default_rng(3).uniform(-1, 1, 63 * 16)
    assert rel(fp.apply_inverse(plan, v), po.pc_apply(v)) <= 1e-12


def test_pc_apply_zero_is_zero():
    op, h, dt = make(1.5, 15, 8)
    plan = fp.build_plan(fp.PreconditionerKind.with_alpha(0.5), 8, dt, op)
    z = fp.apply_inverse(plan, np.zeros(15 * 8))
    assert np.all(z == 0.0)


@pytest.mark.parametrize("gamma,ns,nt,restart", [(1.5, 63, 16, 0), (1.5, 255, 64, 0), (1.5, 1023, 256, 20),
                                                 (1.5, 1023, 256, 5), (1.8, 511, 128, 0), (1.5, 16383, 8, 0)])
def test_gmres_1d(oracle, gamma, ns, nt, restart):
    w = problems.workload_1d(gamma, ns + 1, nt)
    op = fp.AllAtOnceOperator(fp.TimeStencil(nt), fp.RieszJacobian1D(gamma, 1.0, w.h, ns), w.dt)
    plan = fp.build_plan(fp.PreconditionerKind.generalized(), nt, w.dt, op)
    b = problems.rhs(w)
    res = fp.gmres_right(op, plan, b, fp.SolverConfig(tol=1e-10, max_iter=200, restart=restart))
    po = oracle.problem_1d(gamma, 1.0, w.h, ns, nt, w.dt).build_plan()
    xo, ro = po.gmres(b, 1e-10, 200, restart=restart)
    assert res.report.converged and ro.converged
    assert abs(res.report.iterations - ro.iterations) <= 1
    assert rel(res.x, xo) <= 1e-10
    assert res.report.true_relative_residual <= 1e-9


def test_gmres_zero_rhs():
    op, h, dt = make(1.5, 15, 8)
    plan = fp.build_plan(fp.PreconditionerKind.generalized(), 8, dt, op)
    res = fp.gmres_right(op, plan, np.zeros(15 * 8))
    assert res.report.converged and res.report.iterations == 0
    assert np.all(res.x == 0.0)


def test_gmres_budget_exhaustion(oracle):
    op, h, dt = make(1.5, 63, 16)
    plan = fp.build_plan(fp.PreconditionerKind.generalized(), 16, dt, op)
    b = np.random.default_rng(5).uniform(-1, 1, 63 * 16)
    res = fp.gmres_right(op, plan, b, fp.SolverConfig(tol=1e-14, max_iter=3))
    assert not res.report.converged and res.report.iterations == 3
    assert len(res.report.residual_history) == 3


def test_device_tensors_roundtrip(oracle):
    torch = pytest.importorskip("torch")
    op, h, dt = make(1.5, 255, 64)
    plan = fp.build_plan(fp.PreconditionerKind.generalized(), 64, dt, op)
    v = np.random.default_rng(9).uniform(-1, 1, 255 * 64)
    vt = torch.from_numpy(v).cuda()
    y = op.apply(vt)
    op.ctx.synchronize()
    assert rel(y.cpu().numpy(), op.apply(v)) == 0.0
    z = fp.apply_inverse(plan, vt)
    op.ctx.synchronize()
    assert rel(z.cpu().numpy(), fp.apply_inverse(plan, v)) == 0.0


@pytest.mark.parametrize("pinned", [False, True])
def test_gmres_host_buffers_match_device(pinned):
    # host path: upload, solve, x copied back on a side stream while the true-residual check runs
    torch = pytest.importorskip("torch")
    w = problems.workload_1d(1.5, 1024, 64)
    op = fp.AllAtOnceOperator(fp.TimeStencil(64), fp.RieszJacobian1D(1.5, 1.0, w.h, w.n), w.dt)
    plan = fp.build_plan(fp.PreconditionerKind.generalized(), 64, w.dt, op)
    b = problems.rhs(w)
    cfg = fp.SolverConfig(tol=1e-10, max_iter=200, restart=20)
    rd = fp.gmres_right(op, plan, torch.from_numpy(b).cuda(), cfg)
    op.ctx.synchronize()
    if pinned:
        bh = torch.from_numpy(b).pin_memory().numpy()
        xh = torch.empty(b.size, dtype=torch.float64).pin_memory().numpy()
    else:
        bh, xh = b.copy(), np.full(b.size, np.nan)
    for _ in range(2):  # the second call reuses the side stream and the staging buffers
        xh[:] = np.nan
        rh = fp.gmres_right(op, plan, bh, cfg, out=xh)
        assert rh.x is xh
        assert np.array_equal(xh, rd.x.cpu().numpy())
        assert rh.report.iterations == rd.report.iterations
        assert rh.report.true_relative_residual == rd.report.true_relative_residual
    with pytest.raises(ValueError):
        fp.gmres_right(op, plan, bh, cfg, out=np.empty(b.size, dtype=np.float32))


def test_unsupported_sizes_fail_loudly():
    # beyond both the power-of-two kernels and the Bluestein path (n_time <= 4096, n_space <= 2047)
    with pytest.raises(NotImplementedError):
        fp.AllAtOnceOperator(fp.TimeStencil(6), fp.RieszJacobian1D(1.5, 1.0, 1e-4, 9999), 1 / 6)
    with pytest.raises(NotImplementedError):
        fp.AllAtOnceOperator(fp.TimeStencil(5000), fp.RieszJacobian1D(1.5, 1.0, 0.1, 9), 1 / 5000)
    with pytest.raises(ValueError):
        fp.AllAtOnceOperator(fp.TimeStencil(8), fp.RieszJacobian1D(1.5, -1.0, 0.1, 7), 0.1)


@pytest.mark.parametrize("gamma,ns,nt", [(1.9, 7, 8), (1.5, 63, 16), (1.5, 1023, 64), (1.2, 8191, 8),
                                         (1.4, 32767, 4)])
def test_pc_forward_1d(oracle, gamma, ns, nt):
    # apply_forward (alpha_circulant.hpp:212-215) vs the oracle, and the round trip P^{-1} P v = v
    op, h, dt = make(gamma, ns, nt)
    plan = fp.build_plan(fp.PreconditionerKind.with_alpha(0.35), nt, dt, op)
    po = oracle.problem_1d(gamma, 1.0, h, ns, nt, dt).build_plan(0.35)
    v = np.random.default_rng(ns).uniform(-1, 1, ns * nt)
    pv = fp.apply_forward(plan, v)
    assert rel(pv, po.pc_forward(v)) <= 1e-12
    assert rel(fp.apply_inverse(plan, pv), v) <= 1e-10


@pytest.mark.parametrize("gamma,ns,nt", [(1.5, 15, 8), (1.7, 63, 16), (1.5, 1023, 64), (1.2, 8191, 8),
                                         (1.5, 16383, 4), (1.3, 63, 2048), (1.4, 31, 8192)])
def test_full_sweep_1d(oracle, gamma, ns, nt):
    # InnerSweep::full (alpha_circulant.hpp:158-159) vs the oracle's full sweep, and the reference's
    # half == full property (test_pint.cpp:203-216)
    op, h, dt = make(gamma, ns, nt)
    plan = fp.build_plan(fp.PreconditionerKind.generalized(), nt, dt, op)
    po = oracle.problem_1d(gamma, 1.0, h, ns, nt, dt).build_plan()
    v = np.random.default_rng(ns).uniform(-1, 1, ns * nt)
    full = fp.apply_inverse(plan, v, sweep=fp.InnerSweep.full)
    assert rel(full, po.pc_apply(v, True)) <= 1e-12
    # half == full up to rounding; at long series the alpha^{+-k/Nt} scalings amplify it: the oracle's
    # own half-vs-full difference is 6.2e-12 at (1.3, 63, 2048) and 2.1e-11 at (1.4, 31, 8192)
    assert rel(fp.apply_inverse(plan, v), full) <= (1e-12 if nt < 1024 else 2e-11 if nt <= 2048 else 6e-11)
    b = np.random.default_rng(1).uniform(-1, 1, ns * nt)
    r = fp.gmres_right(op, plan, b, fp.SolverConfig(tol=1e-10, sweep=fp.InnerSweep.full))
    xo, ro = po.gmres(b, 1e-10, 200, full_sweep=True)
    assert abs(r.report.iterations - ro.iterations) <= 1 and rel(r.x, xo) <= 1e-10
