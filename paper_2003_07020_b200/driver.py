"""Paper-table path: the reference's manufactured benchmarks and end-to-end driver on the B200 solver.

Mirrors, with the same names and argument meaning:

  Problem1D / Problem2D, example1, example2     problems.hpp:24-131
  Grid1D / Grid2D                               problems.hpp:135-167
  sample_initial / sample_exact / sample_source problems.hpp:169-229
  KrylovMethod, RunConfig, RunResult            driver.hpp:23-45
  run_problem                                   driver.hpp:49-112

The sampling is host setup (numpy, vectorised over the grid); the solve is the device path
(AllAtOnceOperator / build_plan / gmres_right or bicgstab_left of this package).  Closed forms:
the Riesz derivative of a boundary-vanishing symmetric polynomial profile on (0, L) is
-1/(2 cos(gamma pi/2)) sum_p c_p Gamma(p+1)/Gamma(p+1-gamma) (x^{p-gamma} + (L-x)^{p-gamma})
(problems.hpp:44-60).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from enum import Enum
from typing import Callable

import numpy as np

from .solver import (AllAtOnceOperator, InnerSweep, PreconditionerKind, RieszJacobian1D, RieszJacobian2D,
                     SolveReport, SolverConfig, TimeStencil, assemble_rhs, bicgstab_left, build_plan,
                     gmres_right)


def _check_gamma(gamma: float) -> None:
    """problems.hpp:62-65"""
    if not (gamma > 1.0) or gamma > 2.0:
        raise ValueError("benchmark problems require gamma in (1, 2]")


def _reflected_monomial_sum(powers, coeffs, gamma: float, length: float, x: np.ndarray) -> np.ndarray:
    """problems.hpp:47-60: sum_p c_p Gamma(p+1)/Gamma(p+1-gamma) (x^{p-gamma} + (L-x)^{p-gamma})."""
    s = np.zeros_like(x)
    for p, c in zip(powers, coeffs):
        factor = math.gamma(p + 1.0) / math.gamma(p + 1.0 - gamma)
        s = s + c * factor * (np.power(x, p - gamma) + np.power(length - x, p - gamma))
    return s


@dataclass
class Problem1D:
    """problems.hpp:24-32; callables take numpy arrays (x) and a scalar t."""
    gamma: float = 1.5
    kappa: float = 1.0
    a: float = 0.0
    b: float = 1.0
    t_final: float = 1.0
    initial: Callable = None
    source: Callable = None
    exact: Callable = None


@dataclass
class Problem2D:
    """problems.hpp:34-42; callables take numpy arrays (x, y) and a scalar t."""
    gamma_x: float = 1.5
    gamma_y: float = 1.5
    kappa_x: float = 1.0
    kappa_y: float = 1.0
    ax: float = 0.0
    bx: float = 1.0
    ay: float = 0.0
    by: float = 1.0
    t_final: float = 1.0
    initial: Callable = None
    source: Callable = None
    exact: Callable = None


def example1(gamma: float) -> Problem1D:
    """u(x, t) = 15 (1 + gamma/4) e^t x^3 (1-x)^3 on (0, 1), kappa = 0.01 (problems.hpp:69-97)."""
    _check_gamma(gamma)
    kappa = 0.01
    amp = 15.0 * (1.0 + 0.25 * gamma)
    powers, coeffs = (3.0, 4.0, 5.0, 6.0), (1.0, -3.0, 3.0, -1.0)
    riesz_scale = kappa / (2.0 * math.cos(gamma * math.pi / 2.0))

    def exact(x, t):
        w = x * (1.0 - x)
        return amp * math.exp(t) * w * w * w

    def source(x, t):
        return exact(x, t) + amp * math.exp(t) * riesz_scale * _reflected_monomial_sum(powers, coeffs, gamma, 1.0, x)

    return Problem1D(gamma=gamma, kappa=kappa, a=0.0, b=1.0, t_final=1.0, initial=lambda x: exact(x, 0.0),
                     source=source, exact=exact)


def example2(gamma_x: float, gamma_y: float) -> Problem2D:
    """u(x, y, t) = e^{-t/3} x^4 (2-x)^4 y^4 (2-y)^4 on (0, 2)^2, kappa = 0.01 (problems.hpp:101-131)."""
    _check_gamma(gamma_x)
    _check_gamma(gamma_y)
    powers, coeffs = (4.0, 5.0, 6.0, 7.0, 8.0), (16.0, -32.0, 24.0, -8.0, 1.0)
    kx = ky = 0.01
    scale_x = kx / (2.0 * math.cos(gamma_x * math.pi / 2.0))
    scale_y = ky / (2.0 * math.cos(gamma_y * math.pi / 2.0))

    def profile(s):
        w = s * (2.0 - s)
        w2 = w * w
        return w2 * w2

    def exact(x, y, t):
        return math.exp(-t / 3.0) * profile(x) * profile(y)

    def source(x, y, t):
        decay = math.exp(-t / 3.0)
        fx, fy = profile(x), profile(y)
        f = -fx * fy / 3.0
        f = f + scale_x * fy * _reflected_monomial_sum(powers, coeffs, gamma_x, 2.0, x)
        f = f + scale_y * fx * _reflected_monomial_sum(powers, coeffs, gamma_y, 2.0, y)
        return decay * f

    return Problem2D(gamma_x=gamma_x, gamma_y=gamma_y, kappa_x=kx, kappa_y=ky, ax=0.0, bx=2.0, ay=0.0, by=2.0,
                     t_final=2.0, initial=lambda x, y: exact(x, y, 0.0), source=source, exact=exact)


class Grid1D:
    """problems.hpp:135-145: h_inv intervals, n = h_inv - 1 interior points, x_i = a + (i+1) h."""

    def __init__(self, a: float, b: float, h_inv: int):
        if h_inv < 2:
            raise ValueError("Grid1D: need at least 2 intervals")
        self.a, self.h, self.n = float(a), (b - a) / h_inv, int(h_inv) - 1

    def x(self, i=None):
        i = np.arange(self.n) if i is None else i
        return self.a + (i + 1) * self.h


class Grid2D:
    """problems.hpp:147-167: equal extents, lattice index ix * n + iy (x slow)."""

    def __init__(self, ax: float, bx: float, ay: float, by: float, h_inv: int):
        if h_inv < 2:
            raise ValueError("Grid2D: need at least 2 intervals")
        lx, ly = bx - ax, by - ay
        if abs(lx - ly) > 1e-14 * max(abs(lx), abs(ly)):
            raise ValueError("Grid2D: domain must have equal extents in x and y")
        self.ax, self.ay, self.h, self.n_per_dim = float(ax), float(ay), lx / h_inv, int(h_inv) - 1

    def x(self, ix=None):
        ix = np.arange(self.n_per_dim) if ix is None else ix
        return self.ax + (ix + 1) * self.h

    def y(self, iy=None):
        iy = np.arange(self.n_per_dim) if iy is None else iy
        return self.ay + (iy + 1) * self.h

    def index(self, ix: int, iy: int) -> int:
        return ix * self.n_per_dim + iy

    def size(self) -> int:
        return self.n_per_dim * self.n_per_dim

    def mesh(self):
        return np.meshgrid(self.x(), self.y(), indexing="ij")  # [ix, iy] -> ravel = ix * n + iy


def sample_initial(p, g) -> np.ndarray:
    """problems.hpp:169-173 / 195-201"""
    if isinstance(p, Problem1D):
        return np.ascontiguousarray(p.initial(g.x()), dtype=np.float64)
    X, Y = g.mesh()
    return np.ascontiguousarray(p.initial(X, Y).ravel(), dtype=np.float64)


def sample_exact(p, g, t: float) -> np.ndarray:
    """problems.hpp:175-179 / 203-209"""
    if isinstance(p, Problem1D):
        return np.ascontiguousarray(p.exact(g.x(), t), dtype=np.float64)
    X, Y = g.mesh()
    return np.ascontiguousarray(p.exact(X, Y, t).ravel(), dtype=np.float64)


def sample_source(p, g, dt: float, n_time: int) -> np.ndarray:
    """problems.hpp:181-193 / 211-227: f[k * ns + i] = f(x_i, (k+1) dt), time-major."""
    if isinstance(p, Problem1D):
        x = g.x()
        return np.concatenate([p.source(x, (k + 1.0) * dt) for k in range(n_time)]).astype(np.float64)
    X, Y = g.mesh()
    return np.concatenate([p.source(X, Y, (k + 1.0) * dt).ravel() for k in range(n_time)]).astype(np.float64)


class KrylovMethod(Enum):
    """driver.hpp:23"""
    gmres = 0
    bicgstab = 1


@dataclass
class RunConfig:
    """driver.hpp:25-32 (+ restart, the B200 GMRES(m) knob; 0 = the reference's unrestarted GMRES)."""
    n_time: int = 64
    h_inv: int = 128
    kind: PreconditionerKind = field(default_factory=PreconditionerKind.generalized)
    method: KrylovMethod = KrylovMethod.gmres
    solver: SolverConfig = field(default_factory=SolverConfig)
    sweep: InnerSweep = InnerSweep.half


@dataclass
class RunResult:
    """driver.hpp:34-45"""
    n_time: int = 0
    n_space: int = 0
    dof: int = 0
    dt: float = 0.0
    h: float = 0.0
    alpha: float = 0.0
    report: SolveReport = None
    err_inf: float = 0.0
    final_state: np.ndarray = None
    warnings: list = field(default_factory=list)


def _solve_all_at_once(jac, h, t_final, u0, f_flat, exact_final, cfg: RunConfig, context=None) -> RunResult:
    """driver.hpp:49-92 on the device: stencil, operator, rhs, plan, Krylov, err_inf at t_final."""
    nt = cfg.n_time
    ns = jac.dim()
    dt = t_final / nt
    stencil = TimeStencil(nt)
    op = AllAtOnceOperator(stencil, jac, dt, context)
    rhs = assemble_rhs(stencil, dt, f_flat, u0)
    plan = build_plan(cfg.kind, nt, dt, op)
    scfg = SolverConfig(tol=cfg.solver.tol, max_iter=cfg.solver.max_iter, restart=cfg.solver.restart,
                        sweep=cfg.sweep)
    solve = gmres_right if cfg.method == KrylovMethod.gmres else bicgstab_left
    solved = solve(op, plan, rhs, scfg)
    final = np.array(solved.x[nt * ns - ns:], dtype=np.float64)
    return RunResult(n_time=nt, n_space=ns, dof=nt * ns, dt=dt, h=h, alpha=plan.alpha, report=solved.report,
                     err_inf=float(np.max(np.abs(final - exact_final))) if ns else 0.0, final_state=final,
                     warnings=list(plan.warnings))


def run_problem(p, cfg: RunConfig, context=None) -> RunResult:
    """driver.hpp:94-112"""
    if isinstance(p, Problem1D):
        g = Grid1D(p.a, p.b, cfg.h_inv)
        jac = RieszJacobian1D(p.gamma, p.kappa, g.h, g.n)
    elif isinstance(p, Problem2D):
        g = Grid2D(p.ax, p.bx, p.ay, p.by, cfg.h_inv)
        jac = RieszJacobian2D(p.gamma_x, p.gamma_y, p.kappa_x, p.kappa_y, g.h, g.n_per_dim)
    else:
        raise TypeError("run_problem: Problem1D or Problem2D required")
    dt = p.t_final / cfg.n_time
    return _solve_all_at_once(jac, g.h, p.t_final, sample_initial(p, g), sample_source(p, g, dt, cfg.n_time),
                              sample_exact(p, g, p.t_final), cfg, context)
