"""The sharded solver's per-rank CUDA path (fpc_shard_* entry points) at world size 1 on one
B200: must agree with the single-GPU solve (multi-rank communication is covered by
tests/test_dist_gloo.py on CPU; one GPU cannot host NCCL peers)."""
import numpy as np
import pytest

import paper_2003_07020_b200 as fp
from paper_2003_07020_b200 import problems

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("two_dim,ordering", [(False, "reference"), (True, "reference"), (False, "commuted"),
                                             (True, "commuted")])
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


@pytest.mark.parametrize("ordering", ["reference", "commuted"])
def test_sharded_p2p_world1_matches_single_gpu(oracle, ordering):
    # transport="p2p": every exchange is a peer-store kernel (fpc_shard_scatter_p2p) into the
    # IPC-shared receive buffers (at world size 1 the own buffer)
    torch = pytest.importorskip("torch")
    from paper_2003_07020_b200.distributed import CudaShardKernels, ShardedSolver
    w = problems.workload_1d(1.5, 256, 64)
    ctx = fp.Context(0, torch.cuda.current_stream())
    op = fp.AllAtOnceOperator(fp.TimeStencil(w.n_time), fp.RieszJacobian1D(1.5, 1.0, w.h, w.n), w.dt, ctx)
    plan = fp.build_plan(fp.PreconditionerKind.generalized(), w.n_time, w.dt, op, ordering=fp.Ordering[ordering])
    b = problems.rhs(w)
    bt = torch.from_numpy(b).cuda()
    s = ShardedSolver(w.n_time, w.n_space, CudaShardKernels(op, plan), ordering=ordering, transport="p2p")
    rel = lambda a, c: np.linalg.norm(a - c) / np.linalg.norm(c)
    z1 = s.pc_apply(bt)
    z2 = s.pc_apply(2.0 * bt)  # the receive buffers are reused: the first result must survive
    assert rel(z1.cpu().numpy(), fp.apply_inverse(plan, b)) <= 1e-14
    assert rel(z2.cpu().numpy(), 2.0 * z1.cpu().numpy()) <= 1e-14
    x, rep = s.gmres(bt, 1e-10, 200, restart=20)
    ref = fp.gmres_right(op, plan, b, fp.SolverConfig(tol=1e-10, max_iter=200, restart=20))
    assert rep.converged and rep.iterations == ref.report.iterations
    assert rel(x.cpu().numpy(), ref.x) <= 1e-12
    s.close()


@pytest.mark.parametrize("G", [2, 3, 5])
def test_scatter_p2p_layouts_simulated_ranks(G):
    # the four exchanges of the reference ordering with G destination buffers on one device (the
    # simulated ranks' kernels run one after the other and never wait on each other): every receive
    # buffer must equal the consumer layout the NCCL path assembles with all_to_all + cat
    torch = pytest.importorskip("torch")
    from paper_2003_07020_b200.distributed import CudaShardKernels, offsets, split_counts
    nt, ns = 8 * G, 37
    H, nt_loc = nt // 2 + 1, nt // G
    cs, hs = split_counts(ns, G), split_counts(H, G)
    co, ho = offsets(cs), offsets(hs)
    ctx = fp.Context(0, torch.cuda.current_stream())
    op = fp.AllAtOnceOperator(fp.TimeStencil(16), fp.RieszJacobian1D(1.5, 1.0, 1 / 16, 15), 1 / 16, ctx)
    k = CudaShardKernels(op, None)
    rng = np.random.default_rng(G)
    dev = torch.device("cuda", 0)

    def run(srcs, shapes_dst, es, split_cols, off, stride, row_base, col_base, rows_cols):
        dst = [torch.full((int(np.prod(sh)) * es,), np.nan, dtype=torch.float64, device=dev) for sh in shapes_dst]
        for r in range(G):
            rows, cols = rows_cols(r)
            k.scatter_p2p(srcs[r], rows, cols, es, split_cols, [d.data_ptr() for d in dst], off, stride(r),
                          row_base(r), col_base(r))
        torch.cuda.synchronize()
        return [d.cpu().numpy() for d in dst]

    # 1. time -> space: V_r [nt_loc][ns] -> cols_d [nt][cs_d]
    v = rng.standard_normal((nt, ns))
    got = run([torch.from_numpy(v[r * nt_loc:(r + 1) * nt_loc].ravel().copy()).to(dev) for r in range(G)],
              [(nt, cs[d]) for d in range(G)], 1, True, co, lambda r: cs, lambda r: r * nt_loc, lambda r: 0,
              lambda r: (nt_loc, ns))
    for d in range(G):
        assert np.array_equal(got[d], v[:, co[d]:co[d] + cs[d]].ravel())
    # 3. space -> frequency (complex): Z_r [H][cs_r] -> rows_d [hs_d][ns]
    Zc = rng.standard_normal((H, ns)) + 1j * rng.standard_normal((H, ns))
    srcs = [torch.from_numpy(np.ascontiguousarray(Zc[:, co[r]:co[r] + cs[r]]).view(np.float64).ravel().copy()).to(dev)
            for r in range(G)]
    got = run(srcs, [(hs[d], ns) for d in range(G)], 2, False, ho, lambda r: [ns] * G, lambda r: 0,
              lambda r: co[r], lambda r: (H, cs[r]))
    for d in range(G):
        assert np.array_equal(got[d].view(np.complex128), Zc[ho[d]:ho[d] + hs[d]].ravel())
    # 5. frequency -> space (complex): rows_r [hs_r][ns] -> Z_d [H][cs_d]
    srcs = [torch.from_numpy(np.ascontiguousarray(Zc[ho[r]:ho[r] + hs[r]]).view(np.float64).ravel().copy()).to(dev)
            for r in range(G)]
    got = run(srcs, [(H, cs[d]) for d in range(G)], 2, True, co, lambda r: cs, lambda r: ho[r], lambda r: 0,
              lambda r: (hs[r], ns))
    for d in range(G):
        assert np.array_equal(got[d].view(np.complex128), Zc[:, co[d]:co[d] + cs[d]].ravel())
    # 7. space -> time: z_r [nt][cs_r] -> w_d [nt_loc][ns]
    srcs = [torch.from_numpy(np.ascontiguousarray(v[:, co[r]:co[r] + cs[r]]).ravel().copy()).to(dev) for r in range(G)]
    got = run(srcs, [(nt_loc, ns) for d in range(G)], 1, False, [d * nt_loc for d in range(G)], lambda r: [ns] * G,
              lambda r: 0, lambda r: co[r], lambda r: (nt, cs[r]))
    for d in range(G):
        assert np.array_equal(got[d], v[d * nt_loc:(d + 1) * nt_loc].ravel())


_IPC_CHILD = r"""
import sys, ctypes as C, torch
sys.path.insert(0, sys.argv[1])
import paper_2003_07020_b200 as fp
from paper_2003_07020_b200.distributed import CudaShardKernels
ctx = fp.Context(0, torch.cuda.current_stream())
op = fp.AllAtOnceOperator(fp.TimeStencil(16), fp.RieszJacobian1D(1.5, 1.0, 1 / 16, 15), 1 / 16, ctx)
k = CudaShardKernels(op, None)
peer = k.ipc_open(bytes.fromhex(sys.argv[2]))
src = torch.arange(64, dtype=torch.float64, device="cuda") + 0.5
k.scatter_p2p(src, 8, 8, 1, True, [peer], [0], [8], 0, 0)
torch.cuda.synchronize()
k.ipc_close(peer)
print("child ok")
"""


def test_ipc_peer_store_from_another_process(tmp_path):
    # the IPC plumbing of the p2p transport: a second process (same GPU) maps this process's receive
    # buffer and stores into it with the scatter kernel; no kernel of either process waits on the other
    import os
    import subprocess
    import sys
    torch = pytest.importorskip("torch")
    from paper_2003_07020_b200.distributed import CudaShardKernels
    ctx = fp.Context(0, torch.cuda.current_stream())
    op = fp.AllAtOnceOperator(fp.TimeStencil(16), fp.RieszJacobian1D(1.5, 1.0, 1 / 16, 15), 1 / 16, ctx)
    k = CudaShardKernels(op, None)
    ptr = k.alloc_shared(64)
    buf = k.tensor_at(ptr, 64)
    buf.fill_(-1.0)
    torch.cuda.synchronize()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", _IPC_CHILD, root, k.ipc_handle(ptr).hex()],
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "child ok" in out.stdout, out.stderr[-2000:]
    assert np.array_equal(buf.cpu().numpy(), np.arange(64) + 0.5)
    k.free_shared(ptr)
