"""Parity at the BASELINE.json configs themselves (north star: "GPU solutions matching the CPU
oracle ... on all five configs"), GPU solve through the C-ABI against the UNMODIFIED reference
(oracle/_ref, the reference headers compiled by oracle/Makefile; it travels to the GPU box as a
prebuilt .so) on the same seeded inputs.  Not skippable: a missing oracle/_ref is a failure.

  config 0  1D 1023 x 256, gamma 1.5, GMRES(20), tol 1e-10              full size
  config 1  1D 8191 x 2048, gamma 1.2 and 1.8, GMRES(20), tol 1e-10     full size
  config 2  2D 255^2 x 512, gamma 1.3/1.7, GMRES(20), tol 1e-10         full size
  config 3  2D, gamma 1.5/1.5, GMRES(10), tol 1e-9: its exact parameters on a reduced grid (the full
            8.6 GB-per-vector case needs ~190 GB of host RAM for the reference),
            against the restart emulation on the reference's own gmres_right
  config 4  PC apply + matvec sweep: the corner points 65535 x 256 and 1023 x 8192 (and 8191 x
            8192) against the reference's apply_inverse / AllAtOnceOperator::apply

Bars (BASELINE north star): iterations equal +-1, ||x - x_ref|| / ||x_ref|| <= 1e-10.  Config 1 at
gamma 1.8 is the exception: there the reference's own x is only accurate to its true relative
residual (2.6e-8), so that case asserts equal iterations, a true residual no worse than the
reference's, and a distance below the reference's own residual (see the test's docstring).
"""
import os

import numpy as np
import pytest

import paper_2003_07020_b200 as fp
from paper_2003_07020_b200 import problems

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def ref():
    from oracle import oracle as O
    assert O.Reference.available(), (
        "oracle/_ref/libfracpint_ref.so is missing: build it with `make -C oracle` where "
        "/root/reference exists (it is shipped prebuilt to the GPU box)")
    r = O.Reference()
    r.set_threads(os.cpu_count() or 1)
    return r


def gpu_problem(w):
    if w.two_dim:
        jac = fp.RieszJacobian2D(w.gamma[0], w.gamma[1], 1.0, 1.0, w.h, w.n)
    else:
        jac = fp.RieszJacobian1D(w.gamma[0], 1.0, w.h, w.n)
    op = fp.AllAtOnceOperator(fp.TimeStencil(w.n_time), jac, w.dt)
    plan = fp.build_plan(fp.PreconditionerKind.generalized(), w.n_time, w.dt, op)
    return op, plan


def ref_problem(backend, w):
    if w.two_dim:
        p = backend.problem_2d(w.gamma[0], w.gamma[1], 1.0, 1.0, w.h, w.n, w.n_time, w.dt)
    else:
        p = backend.problem_1d(w.gamma[0], 1.0, w.h, w.n, w.n_time, w.dt)
    return p.build_plan()


def solve_both(ref, w):
    op, plan = gpu_problem(w)
    b = problems.rhs(w)
    res = fp.gmres_right(op, plan, b, fp.SolverConfig(tol=w.tol, max_iter=200, restart=w.restart))
    pr = ref_problem(ref, w)
    # the reference has no restart; configs 0-2 converge in fewer than `restart` steps, where
    # GMRES(20) and the reference's unrestarted gmres_right are the same iteration
    xr, rr = pr.gmres(b, w.tol, 200)
    assert rr.iterations < w.restart
    return res, xr, rr


@pytest.mark.parametrize("cfg", [(0, None), (1, 1.2), (2, None)],
                         ids=["cfg0_1d_1023x256", "cfg1_1d_8191x2048_g1.2", "cfg2_2d_255sq_x512"])
def test_config_solve_vs_reference(ref, cfg):
    w = problems.config(cfg[0], cfg[1])
    res, xr, rr = solve_both(ref, w)
    print(f"\n{w.name}: iterations gpu {res.report.iterations} ref {rr.iterations}; x vs ref {rel(res.x, xr):.3e}; "
          f"TRR gpu {res.report.true_relative_residual:.3e} ref {rr.true_relative_residual:.3e}; ref {rr.seconds:.1f} s")
    assert res.report.converged and rr.converged
    assert abs(res.report.iterations - rr.iterations) <= 1, (res.report.iterations, rr.iterations)
    assert rel(res.x, xr) <= 1e-10, rel(res.x, xr)
    # residual histories agree to well within the straddle of tol (~10x)
    h_gpu, h_ref = np.array(res.report.residual_history), np.array(rr.residual_history)
    m = min(len(h_gpu), len(h_ref))
    assert np.all(np.abs(np.log10(h_gpu[:m] / h_ref[:m])) < 0.05)


def test_config1_gamma18_conditioning_floor(ref):
    """Config 1, gamma 1.8: the reference's own solution is only as accurate as its true relative
    residual, 2.6e-8 -- 260x the tolerance (it stops on the recurrence
    residual, which the alpha^{-k/Nt} scalings (1/alpha = 4096) decouple from ||b - A x||).  Two
    solutions x, y with residuals r_x, r_y differ by at most ||A^-1|| (||r_x|| + ||r_y||), so the
    1e-10 bar on ||x_gpu - x_ref|| is below what the reference's x itself resolves.  Asserted here:
    the same iteration count, a GPU true residual no worse than the reference's, and a distance
    to the reference's x below the reference's own true residual (and within 1e-9)."""
    w = problems.config(1, 1.8)
    res, xr, rr = solve_both(ref, w)
    d_gpu = rel(res.x, xr)
    print(f"\n{w.name}: iterations gpu {res.report.iterations} ref {rr.iterations}; x gpu-ref {d_gpu:.3e}; "
          f"TRR gpu {res.report.true_relative_residual:.3e} ref {rr.true_relative_residual:.3e}")
    assert res.report.converged and rr.converged
    assert res.report.iterations == rr.iterations
    assert res.report.true_relative_residual <= rr.true_relative_residual
    assert d_gpu <= min(rr.true_relative_residual, 1e-9), (d_gpu, rr.true_relative_residual)


@pytest.mark.parametrize("n,nt", [(255, 1024), (511, 128), (1023, 16)],
                         ids=["255sq_x1024", "511sq_x128", "1023sq_x16"])
def test_config3_parameters_reduced_grid(ref, n, nt):
    """Config 3's solver parameters exactly (gamma 1.5/1.5, kappa 1, GMRES(10), tol 1e-9, seeded
    source and u0 as config 3) on the largest grids the reference finishes in about a minute on the
    box, against GMRES(10) emulated on the reference's own gmres_right.  1023^2 x 16
    is config 3's own lattice (the one-warp-per-row 1024-point kernels, kernels_warp32.cu) on a
    short time axis."""
    w = problems.workload_2d(1.5, 1.5, n + 1, nt, tol=1e-9, restart=10)
    op, plan = gpu_problem(w)
    b = problems.rhs(w)
    res = fp.gmres_right(op, plan, b, fp.SolverConfig(tol=w.tol, max_iter=200, restart=10))
    xr, rr = ref_problem(ref, w).gmres_restarted(b, w.tol, 200, 10)
    print(f"\n{w.name} GMRES(10): iterations gpu {res.report.iterations} (restarts {res.report.restarts}) ref "
          f"{rr['iterations']} (restarts {rr['restarts']}); x vs ref {rel(res.x, xr):.3e}; TRR gpu "
          f"{res.report.true_relative_residual:.3e} ref {rr['true_relative_residual']:.3e}; ref {rr['seconds']:.1f} s")
    assert res.report.converged and rr["converged"]
    assert abs(res.report.iterations - rr["iterations"]) <= 1, (res.report.iterations, rr["iterations"])
    assert rel(res.x, xr) <= 1e-10, rel(res.x, xr)
    assert res.report.true_relative_residual <= 1e-8


@pytest.mark.parametrize("nx,nt", [(65535, 256), (1023, 8192), (8191, 8192)])
def test_config4_corner_points(ref, nx, nt):
    """Config 4 (gamma 1.5, kappa 1, alpha = dt/2): complex128 seeded Gaussian input = a batch of two
    real vectors (Re, Im) since the operators are real-linear; PC apply and matvec
    against the reference's apply_inverse / AllAtOnceOperator::apply."""
    h, dt = 1.0 / (nx + 1), 1.0 / nt
    op = fp.AllAtOnceOperator(fp.TimeStencil(nt), fp.RieszJacobian1D(1.5, 1.0, h, nx), dt)
    plan = fp.build_plan(fp.PreconditionerKind.generalized(), nt, dt, op)
    pr = ref.problem_1d(1.5, 1.0, h, nx, nt, dt).build_plan()
    g = np.random.default_rng(20260819 + nx * 131 + nt)
    z = g.standard_normal(nx * nt) + 1j * g.standard_normal(nx * nt)
    for part in (z.real.copy(), z.imag.copy()):
        print(f"\ncfg4 {nx}x{nt}: pc vs ref {rel(fp.apply_inverse(plan, part), pr.pc_apply(part)):.3e} "
              f"matvec vs ref {rel(op.apply(part), pr.matvec(part)):.3e}")
        # the host setup (tau spectrum, lambda, scalings) is the reference's to the bit
        # (tests/test_abi.py), so what remains is FFT rounding amplified by the alpha^{-k/Nt}
        # scalings (1/alpha = 2 Nt): 1e-12, and 1e-11 at Nt = 8192
        assert rel(fp.apply_inverse(plan, part), pr.pc_apply(part)) <= (1e-11 if nt >= 8192 else 1e-12)
        assert rel(op.apply(part), pr.matvec(part)) <= 1e-13


@pytest.mark.parametrize("cfg", [(1, 1.2), (2, None), (3, None)], ids=["cfg1", "cfg2", "cfg3"])
def test_full_size_properties(cfg):
    """Size-independent properties at the BASELINE sizes themselves (config 3: 8.6 GB vectors, which
    no CPU oracle here can hold): real-linearity of the matvec and of P^{-1}, the round trip
    P (P^{-1} v) = v (test_pint.cpp:188-201), and P^{-1} of a PC image, all device-resident."""
    torch = pytest.importorskip("torch")
    w = problems.config(cfg[0], cfg[1])
    op, plan = gpu_problem(w)
    n = w.dim
    g = torch.Generator(device="cuda")
    g.manual_seed(20260819 + cfg[0])
    u = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    v = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    a, b = 0.75, -1.25
    nrm = lambda t: float(torch.linalg.vector_norm(t))
    # linearity of A
    s = a * u + b * v
    As = op.apply(s)
    Au, Av = op.apply(u), op.apply(v)
    lin = nrm(As - (a * Au + b * Av)) / nrm(As)
    del As, Au, Av
    # linearity of P^{-1} and the round trip
    Ps = fp.apply_inverse(plan, s)
    Pu = fp.apply_inverse(plan, u)
    Pv = fp.apply_inverse(plan, v)
    lin_p = nrm(Ps - (a * Pu + b * Pv)) / nrm(Ps)
    del Pu, Pv, Ps
    z = fp.apply_inverse(plan, u)
    back = fp.apply_forward(plan, z)
    rt = nrm(back - u) / nrm(u)
    op.ctx.synchronize()
    print(f"\n{w.name}: A linearity {lin:.2e}, P^-1 linearity {lin_p:.2e}, P P^-1 u - u {rt:.2e}")
    assert lin <= 1e-13 and lin_p <= 1e-12
    # the round trip loses what the alpha^{-k/Nt} scalings amplify (1/alpha = 2 Nt)
    assert rt <= 1e-13 * 2 * w.n_time
