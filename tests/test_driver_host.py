"""Paper-table path, host side (CPU): the manufactured benchmarks' sampling and all-at-once rhs
(paper_2003_07020_b200/driver.py) against what the reference's own run_problem assembled
(tests/golden rp* fixtures, driver.hpp:49-112 / problems.hpp:69-229), plus the argument checks the
reference throws on."""
import os

import numpy as np
import pytest

from paper_2003_07020_b200 import driver as D
from paper_2003_07020_b200.solver import TimeStencil, assemble_rhs

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "fracpint_ref_golden.npz")


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def problem_and_grid(prm):
    dim, gx, gy, nt, h_inv = prm[:5]
    if int(dim) == 1:
        p = D.example1(gx)
        return p, D.Grid1D(p.a, p.b, int(h_inv)), int(nt)
    p = D.example2(gx, gy)
    return p, D.Grid2D(p.ax, p.bx, p.ay, p.by, int(h_inv)), int(nt)


@pytest.mark.parametrize("tag", ["rp1a", "rp1d", "rp2a"])
def test_rhs_matches_reference(gold, tag):
    p, g, nt = problem_and_grid(gold[f"{tag}_params"])
    dt = p.t_final / nt
    f = D.sample_source(p, g, dt, nt)
    u0 = D.sample_initial(p, g)
    b = assemble_rhs(TimeStencil(nt), dt, f, u0)
    ref = gold[f"{tag}_rhs"]
    assert b.shape == ref.shape
    # libm pow/tgamma vs numpy: a few ulps on each source sample
    assert np.abs(b - ref).max() <= 1e-13 * np.abs(ref).max()


@pytest.mark.parametrize("tag", ["rp1a", "rp1c", "rp2b", "rp2d"])
def test_exact_final_matches_reference(gold, tag):
    p, g, _ = problem_and_grid(gold[f"{tag}_params"])
    ex = D.sample_exact(p, g, p.t_final)
    assert np.abs(ex - gold[f"{tag}_exact"]).max() <= 1e-14 * np.abs(gold[f"{tag}_exact"]).max()


def test_grid_and_problem_errors():
    # problems.hpp:62-65, 138, 152-156
    with pytest.raises(ValueError):
        D.example1(1.0)
    with pytest.raises(ValueError):
        D.example2(1.5, 2.5)
    with pytest.raises(ValueError):
        D.Grid1D(0, 1, 1)
    with pytest.raises(ValueError):
        D.Grid2D(0, 1, 0, 2, 8)
    g = D.Grid2D(0, 2, 0, 2, 8)
    assert g.index(2, 3) == 2 * 7 + 3 and g.size() == 49 and g.h == 0.25
    g1 = D.Grid1D(0, 1, 4)
    assert np.allclose(g1.x(), [0.25, 0.5, 0.75])


def test_example_closed_forms():
    # example1 exact at t=0 is the initial condition; the source includes u_t = u
    p = D.example1(1.5)
    x = np.linspace(0.1, 0.9, 5)
    assert np.allclose(p.initial(x), 15 * (1 + 1.5 / 4) * (x * (1 - x)) ** 3)
    q = D.example2(1.5, 1.5)
    X, Y = np.meshgrid(x, x, indexing="ij")
    assert np.allclose(q.exact(X, Y, 3.0), np.exp(-1.0) * (X * (2 - X)) ** 4 * (Y * (2 - Y)) ** 4)
