"""The sharded solver's per-rank CUDA path (fpc_shard_* entry points) at world size 1 on one
B200: must agree with the single-GPU solve (multi-rank communication is covered by
tests/test_dist_gloo.py on CPU; one GPU cannot host NCCL peers)."""
import numpy as np
import pytest

import paper_2003_07020_b200 as fp
from paper_2003_07020_b200 import problems

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("two_dim,ordering", [(False, "reference"), (True, "reference"), (False, "commuted")])
def test_sharded_world1_matches_single_gpu(oracle, two_dim, ordering):
    torch = pytest.importorskip("torch")
    from paper_2003_07020_b200.distributed import CudaShardKernels, ShardedSolver
    if two_dim:
        w = problems.workload_2d(1.3, 1.7, 32, 16)
        jac = fp.RieszJacobian2D(1.3, 1.7, 1.0, 1.0, w.h, w.n)
    else:
        w = problems.workload_1d(1.5, 256, 64)
        jac = fp.RieszJacobian1D(1.5, 1.0, w.h, w.n)
    ctx = fp.Context(0, torch.cuda.current_stream())
    op = fp.AllAtOnceOperator(fp.TimeStencil(w.n_time), jac, w.dt, ctx)
    plan = fp.build_plan(fp.PreconditionerKind.generalized(), w.n_time, w.dt, op,
                         ordering=fp.Ordering[ordering])
    b = problems.rhs(w)
    bt = torch.from_numpy(b).cuda()
    s = ShardedSolver(w.n_time, w.n_space, CudaShardKernels(op, plan), ordering=ordering)
    rel = lambda a, c: np.linalg.norm(a - c) / np.linalg.norm(c)
    assert rel(s.matvec(bt).cpu().numpy(), op.apply(b)) <= 1e-14
    assert rel(s.pc_apply(bt).cpu().numpy(), fp.apply_inverse(plan, b)) <= 1e-14
    x, rep = s.gmres(bt, 1e-10, 200, restart=20)
    ref = fp.gmres_right(op, plan, b, fp.SolverConfig(tol=1e-10, max_iter=200, restart=20))
    assert rep.converged and rep.iterations == ref.report.iterations
    assert rel(x.cpu().numpy(), ref.x) <= 1e-12
    assert rep.true_relative_residual <= 1e-9
