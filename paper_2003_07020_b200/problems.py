"""Grids and the seeded BASELINE workloads (problems.hpp:133-222 grids/samplers; BASELINE.json
configs 0-4 with seeded sources instead of the manufactured examples -- SURVEY §8(d)).

Inputs are generated on the host once (numpy PCG64, seed recorded) and fed to both the oracle
and the GPU, so RNG differences cannot break parity.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Grid1D:
    """problems.hpp:135-146: h = (b-a)/h_inv, n = h_inv - 1, x_i = a + (i+1) h."""
    a: float
    b: float
    h_inv: int

    def __post_init__(self):
        if self.h_inv < 2:
            raise ValueError("Grid1D: need at least 2 intervals")
        self.h = (self.b - self.a) / self.h_inv
        self.n = self.h_inv - 1

    def x(self) -> np.ndarray:
        return self.a + (np.arange(self.n) + 1) * self.h


@dataclass
class Grid2D:
    """problems.hpp:148-167: lattice index ix*n + iy (x slow)."""
    ax: float
    bx: float
    ay: float
    by: float
    h_inv: int

    def __post_init__(self):
        if self.h_inv < 2:
            raise ValueError("Grid2D: need at least 2 intervals")
        lx, ly = self.bx - self.ax, self.by - self.ay
        if abs(lx - ly) > 1e-14 * max(abs(lx), abs(ly)):
            raise ValueError("Grid2D: domain must have equal extents in x and y")
        self.h = lx / self.h_inv
        self.n_per_dim = self.h_inv - 1

    def x(self) -> np.ndarray:
        return self.ax + (np.arange(self.n_per_dim) + 1) * self.h

    def y(self) -> np.ndarray:
        return self.ay + (np.arange(self.n_per_dim) + 1) * self.h


@dataclass
class Workload:
    name: str
    two_dim: bool
    gamma: tuple
    kappa: tuple
    h: float
    n: int            # 1D: n_space; 2D: n per dim
    n_time: int
    dt: float
    tol: float
    restart: int
    u0: np.ndarray
    f: np.ndarray
    seed: int

    @property
    def n_space(self) -> int:
        return self.n * self.n if self.two_dim else self.n

    @property
    def dim(self) -> int:
        return self.n_space * self.n_time


def _src(seed: int, count: int) -> np.ndarray:
    return np.random.default_rng(seed).uniform(-1.0, 1.0, count)


def workload_1d(gamma: float, h_inv: int, n_time: int, seed: int = 20260819, tol: float = 1e-10,
                restart: int = 20, name: str = "") -> Workload:
    """Configs 0/1: (0,1), kappa=1, T=1, u0 = x^2(1-x)^2, f ~ U[-1,1] seeded."""
    g = Grid1D(0.0, 1.0, h_inv)
    x = g.x()
    u0 = x ** 2 * (1 - x) ** 2
    return Workload(name or f"1d_g{gamma}_n{g.n}_t{n_time}", False, (gamma,), (1.0,), g.h, g.n, n_time,
                    1.0 / n_time, tol, restart, u0, _src(seed, g.n * n_time), seed)


def workload_2d(gamma_x: float, gamma_y: float, h_inv: int, n_time: int, seed: int = 20260819,
                tol: float = 1e-10, restart: int = 20, name: str = "") -> Workload:
    """Configs 2/3: (0,1)^2, kappa=1, u0 = x^2(1-x)^2 y^2(1-y)^2, seeded f."""
    g = Grid2D(0.0, 1.0, 0.0, 1.0, h_inv)
    x, y = g.x(), g.y()
    px = x ** 2 * (1 - x) ** 2
    py = y ** 2 * (1 - y) ** 2
    u0 = np.outer(px, py).ravel()
    n = g.n_per_dim
    return Workload(name or f"2d_g{gamma_x},{gamma_y}_n{n}_t{n_time}", True, (gamma_x, gamma_y), (1.0, 1.0),
                    g.h, n, n_time, 1.0 / n_time, tol, restart, u0, _src(seed, n * n * n_time), seed)


# BASELINE.json configs
def config(idx: int, gamma: float | None = None) -> Workload:
    if idx == 0:
        return workload_1d(1.5, 1024, 256, tol=1e-10, restart=20, name="cfg0_1d_1023x256_g1.5")
    if idx == 1:
        g = 1.2 if gamma is None else gamma
        return workload_1d(g, 8192, 2048, tol=1e-10, restart=20, name=f"cfg1_1d_8191x2048_g{g}")
    if idx == 2:
        return workload_2d(1.3, 1.7, 256, 512, tol=1e-10, restart=20, name="cfg2_2d_255sq_x512_g1.3_1.7")
    if idx == 3:
        return workload_2d(1.5, 1.5, 1024, 1024, tol=1e-9, restart=10, name="cfg3_2d_1023sq_x1024_g1.5")
    raise ValueError("configs 0-3 are solves; config 4 is the apply sweep (bench.py --sweep)")


def rhs(w: Workload) -> np.ndarray:
    """b = assemble_rhs(stencil, dt, f, u0) (all_at_once.hpp:66-80), in numpy."""
    ns = w.n_space
    b = w.dt * w.f
    b[:ns] += w.u0
    b[ns:2 * ns] -= 0.5 * w.u0
    return b
