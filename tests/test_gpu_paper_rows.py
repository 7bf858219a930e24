"""Paper-table path on the B200 (driver.run_problem over the manufactured benchmarks).

1. The reference's own acceptance rows, restated from acceptance.cpp:227-272 (the paper's tables:
   iterations within +/-2 for the adaptive alpha and for alpha = 1, max-norm error within 1%).
2. The golden rp* fixtures the reference's run_problem produced (tests/golden/make_golden.py):
   iterations within +/-1 (BiCGSTAB counts halves), err_inf and the final state to rounding."""
import os

import numpy as np
import pytest

import paper_2003_07020_b200 as fp
from paper_2003_07020_b200 import driver as D

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "fracpint_ref_golden.npz")


def run_row(p, nt, h_inv, method):
    """acceptance.cpp:161-176"""
    cfg = D.RunConfig(n_time=nt, h_inv=h_inv, method=method, kind=fp.PreconditionerKind.generalized())
    ra = D.run_problem(p, cfg)
    cfg.kind = fp.PreconditionerKind.strang()
    r1 = D.run_problem(p, cfg)
    return ra.report.iterations, r1.report.iterations, ra.err_inf, ra.report.converged and r1.report.converged


# acceptance.cpp:227-247: (gamma, nt, 1/h, iters alpha, iters alpha=1, err)
ROWS_1D = [
    (1.2, 64, 128, 7, 19, 9.7599e-5), (1.2, 64, 256, 7, 19, 9.4838e-5), (1.2, 64, 512, 8, 19, 9.4147e-5),
    (1.2, 64, 1024, 8, 19, 9.3974e-5), (1.2, 256, 128, 7, 19, 9.5721e-6), (1.2, 256, 256, 7, 19, 6.8110e-6),
    (1.2, 256, 512, 7, 19, 6.1205e-6), (1.2, 256, 1024, 8, 19, 5.9481e-6),
    (1.5, 64, 128, 8, 15, 1.0514e-4), (1.9, 64, 128, 7, 11, 1.2052e-4),
]
# acceptance.cpp:250-272: 2D rows nt = 64, 1/h = 64, BiCGSTAB
ROWS_2D = [(1.4, 1.2, 4.0, 12.0, 1.2627e-4), (1.5, 1.5, 4.0, 11.0, 1.5758e-4), (1.7, 1.9, 4.0, 11.5, 2.3321e-4)]


@pytest.mark.parametrize("row", ROWS_1D)
def test_paper_rows_1d(row):
    gamma, nt, h_inv, it_a, it_1, err = row
    ia, i1, e, conv = run_row(D.example1(gamma), nt, h_inv, D.KrylovMethod.gmres)
    assert conv
    assert abs(ia - it_a) <= 2 and abs(i1 - it_1) <= 2
    assert abs(e - err) <= 1e-2 * err


@pytest.mark.parametrize("row", ROWS_2D)
def test_paper_rows_2d(row):
    gx, gy, it_a, it_1, err = row
    ia, i1, e, conv = run_row(D.example2(gx, gy), 64, 64, D.KrylovMethod.bicgstab)
    assert conv
    assert abs(ia - it_a) <= 2 and abs(i1 - it_1) <= 2
    assert abs(e - err) <= 1e-2 * err


@pytest.mark.parametrize("tag", ["rp1a", "rp1b", "rp1c", "rp1d", "rp2a", "rp2b", "rp2c", "rp2d"])
def test_run_problem_vs_reference_golden(tag):
    g = np.load(GOLD)
    dim, gx, gy, nt, h_inv, method, strang = g[f"{tag}_params"]
    p = D.example1(gx) if int(dim) == 1 else D.example2(gx, gy)
    cfg = D.RunConfig(n_time=int(nt), h_inv=int(h_inv),
                      method=D.KrylovMethod.bicgstab if int(method) else D.KrylovMethod.gmres,
                      kind=fp.PreconditionerKind.strang() if int(strang) else fp.PreconditionerKind.generalized())
    r = D.run_problem(p, cfg)
    iters, conv, err = g[f"{tag}_result"]
    assert r.report.converged == bool(conv)
    assert abs(r.report.iterations - iters) <= 1.0
    fin = g[f"{tag}_final"]
    # tol 1e-9 solves: the discrete solutions agree to the solver tolerance, far below the
    # discretisation error err_inf measures
    assert np.linalg.norm(r.final_state - fin) <= 1e-7 * np.linalg.norm(fin)
    assert abs(r.err_inf - err) <= 1e-4 * err
    assert r.n_space == (int(h_inv) - 1) ** int(dim) and r.dof == r.n_space * int(nt)
