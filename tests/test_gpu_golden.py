"""GPU path vs the reference's own outputs (tests/golden, produced by the unmodified reference
compiled into oracle/_ref).  Sizes the B200 kernels support (n_space + 1 and n_time powers of two);
p1a..p2c cover 1D/2D, generalized and custom alpha, anisotropic kappa."""
import os

import numpy as np
import pytest

import paper_2003_07020_b200 as fp

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "fracpint_ref_golden.npz")
TAGS = ["p1a", "p1b", "p1c", "p1d", "p2a", "p2b", "p2c", "p1s", "p2s"]  # p?s: Strang alpha = 1


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def make(prm):
    dim, g0, g1, k0, k1, h, n, nt, dt, alpha = prm
    st = fp.TimeStencil(int(nt))
    if int(dim) == 1:
        jac = fp.RieszJacobian1D(g0, k0, h, int(n))
    else:
        jac = fp.RieszJacobian2D(g0, g1, k0, k1, h, int(n))
    op = fp.AllAtOnceOperator(st, jac, dt)
    kind = fp.PreconditionerKind.generalized() if alpha <= 0 else fp.PreconditionerKind.with_alpha(alpha)
    return op, fp.build_plan(kind, int(nt), dt, op)


@pytest.mark.parametrize("tag", TAGS)
def test_gpu_vs_reference_golden(gold, tag):
    op, plan = make(gold[f"{tag}_params"])
    v = gold[f"{tag}_v"]
    a, m = gold[f"{tag}_alpha_margin"]
    assert plan.alpha == a and abs(plan.min_shift_margin - m) <= 1e-11 * m
    assert rel(op.tau_sigma(), gold[f"{tag}_sigma"]) <= 1e-13
    assert rel(op.apply(v), gold[f"{tag}_matvec"]) <= 1e-13
    assert rel(fp.apply_inverse(plan, v), gold[f"{tag}_pc_half"]) <= 1e-11
    res = fp.gmres_right(op, plan, gold[f"{tag}_b"], fp.SolverConfig(tol=1e-10, max_iter=200))
    assert abs(res.report.iterations - int(gold[f"{tag}_iters"][0])) <= 1
    assert rel(res.x, gold[f"{tag}_x"]) <= 1e-10
    h = np.array(res.report.residual_history)
    g = gold[f"{tag}_history"]
    k = min(len(h), len(g))
    assert np.allclose(h[:k], g[:k], rtol=1e-6, atol=1e-13)


@pytest.mark.parametrize("tag", TAGS)
def test_gpu_bicgstab_vs_reference_golden(gold, tag):
    """bicgstab_left (krylov.hpp:204-280) on the device vs the reference's own solve."""
    op, plan = make(gold[f"{tag}_params"])
    res = fp.bicgstab_left(op, plan, gold[f"{tag}_b"], fp.SolverConfig(tol=1e-10, max_iter=200))
    assert res.report.converged
    assert abs(res.report.iterations - float(gold[f"{tag}_bicg_iters"][0])) <= 1.0
    assert rel(res.x, gold[f"{tag}_bicg_x"]) <= 1e-10
    assert res.report.true_relative_residual <= 10 * max(float(gold[f"{tag}_bicg_trr"][0]), 1e-11)
