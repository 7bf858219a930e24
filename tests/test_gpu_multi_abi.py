"""The single-process multi-device solve behind the C-ABI (fpc_multi_* / fpc_sharded_*, SURVEY
§8(b)/(e)).  The box has one GPU, so the rank schedules G = 2, 4 (and 8 in 1D) run with every rank on
device 0 -- the same peer-store kernels, halo copies and event ordering as on G devices, and no kernel
ever waits on another rank.  Checked against the single-device library path and the C oracle."""
import numpy as np
import pytest

import paper_2003_07020_b200 as fp
from paper_2003_07020_b200 import problems

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def build(G, two_dim, n, nt):
    if two_dim:
        w = problems.workload_2d(1.3, 1.7, n + 1, nt)
        jac = fp.RieszJacobian2D(1.3, 1.7, 1.0, 1.0, w.h, n)
    else:
        w = problems.workload_1d(1.5, n + 1, nt)
        jac = fp.RieszJacobian1D(1.5, 1.0, w.h, n)
    md = fp.MultiDevice([0] * G)
    sp = fp.ShardedProblem(md, fp.TimeStencil(nt), jac, w.dt)
    op = fp.AllAtOnceOperator(fp.TimeStencil(nt), jac, w.dt)
    plan = fp.build_plan(fp.PreconditionerKind.generalized(), nt, w.dt, op)
    return w, md, sp, op, plan


@pytest.mark.parametrize("G,two_dim,n,nt", [(1, False, 255, 64), (2, False, 255, 64), (4, False, 1023, 256),
                                            (8, False, 127, 32),
                                            (2, True, 31, 16), (4, True, 63, 32),
                                            # the one-warp-per-transform kernels on shards: n = 1023 rows /
                                            # columns (kernels_warp32.cu), n_time = 1024 on 4096-column
                                            # blocks (kernels_time_warp.cu)
                                            (2, True, 1023, 8), (2, False, 1023, 4096), (2, False, 8191, 1024)])
def test_sharded_operators_match_single_device(G, two_dim, n, nt):
    w, md, sp, op, plan = build(G, two_dim, n, nt)
    v = np.random.default_rng(G * 7 + n).uniform(-1, 1, op.dim())
    assert rel(sp.matvec(v), op.apply(v)) <= 1e-14
    assert rel(sp.apply_inverse(v), fp.apply_inverse(plan, v)) <= 1e-13


@pytest.mark.parametrize("G,two_dim,n,nt,restart", [(2, False, 1023, 256, 20), (4, False, 255, 64, 5),
                                                    (2, True, 63, 32, 0), (4, True, 31, 16, 10)])
def test_sharded_gmres_vs_oracle(oracle, G, two_dim, n, nt, restart):
    w, md, sp, op, plan = build(G, two_dim, n, nt)
    b = problems.rhs(w)
    res = sp.gmres_right(b, fp.SolverConfig(tol=1e-10, max_iter=200, restart=restart))
    po = (oracle.problem_2d(1.3, 1.7, 1, 1, w.h, n, nt, w.dt) if two_dim
          else oracle.problem_1d(1.5, 1.0, w.h, n, nt, w.dt)).build_plan()
    xo, ro = po.gmres(b, 1e-10, 200, restart=restart)
    single = fp.gmres_right(op, plan, b, fp.SolverConfig(tol=1e-10, max_iter=200, restart=restart))
    assert res.report.converged
    assert abs(res.report.iterations - ro.iterations) <= 1
    assert abs(res.report.iterations - single.report.iterations) <= 1
    assert rel(res.x, xo) <= 1e-10 and rel(res.x, single.x) <= 1e-10
    assert res.report.true_relative_residual <= 1e-9


def test_sharded_rejects_bad_layouts():
    md = fp.MultiDevice([0, 0, 0])
    with pytest.raises(ValueError):  # 64 levels over 3 ranks
        fp.ShardedProblem(md, fp.TimeStencil(64), fp.RieszJacobian1D(1.5, 1.0, 1 / 64, 63), 1 / 64)
    with pytest.raises(ValueError):
        fp.MultiDevice([0] * 9)
