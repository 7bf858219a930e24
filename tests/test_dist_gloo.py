"""The frequency-sharded multi-rank solve (paper_2003_07020_b200.distributed) under gloo with
world_size 2 on CPU: layouts, all-to-alls, the BDF2 halo and the reduced Gram-Schmidt must
reproduce the single-process oracle (numpy shard kernels stand in for the CUDA ones)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from dist_cpu_kernels import NumpyShardKernels
    from oracle.oracle import Oracle
    from paper_2003_07020_b200.distributed import ShardedSolver
    two_dim, g, n, nt, restart = case[:5]
    ordering = case[5] if len(case) > 5 else "reference"
    dt = 1.0 / nt
    o = Oracle()
    if two_dim:
        po = o.problem_2d(g[0], g[1], 1.0, 1.0, 1.0 / (n + 1), n, nt, dt).build_plan()
        ns = n * n
        po.scales = (1.0 * (n + 1) ** g[0], 1.0 * (n + 1) ** g[1])  # kappa/h^gamma
    else:
        po = o.problem_1d(g[0], 1.0, 1.0 / (n + 1), n, nt, dt).build_plan()
        ns = n
    k = NumpyShardKernels(po, nt, dt, two_dim, n)
    s = ShardedSolver(nt, ns, k, ordering=ordering)
    rng = np.random.default_rng(5)
    v = rng.uniform(-1, 1, nt * ns)
    lo, hi = s.koff * ns, (s.koff + s.nt_loc) * ns
    vl = torch.from_numpy(v[lo:hi].copy())
    y = s.matvec(vl).numpy()
    z = s.pc_apply(vl).numpy()
    pf = s.pc_apply(vl, forward=True).numpy()
    x, rep = s.gmres(vl, 1e-10, 200, restart)
    res = dict(y=y, z=z, pf=pf, x=x.numpy(), iters=rep.iterations, trr=rep.true_relative_residual)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), **res)
    dist.destroy_process_group()


@pytest.mark.parametrize("case", [(False, (1.5,), 31, 16, 0), (False, (1.3,), 63, 8, 5),
                                  (True, (1.3, 1.7), 7, 8, 0),
                                  (False, (1.5,), 31, 16, 0, "commuted"), (False, (1.7,), 15, 32, 5, "commuted"),
                                  (True, (1.3, 1.7), 7, 8, 0, "commuted")])
def test_sharded_solve_matches_oracle(tmp_path, oracle, case):
    _run_and_check(tmp_path, oracle, case, 2)


@pytest.mark.parametrize("case", [(False, (1.5,), 31, 16, 0), (True, (1.3, 1.7), 7, 8, 0, "commuted"),
                                  (False, (1.7,), 15, 32, 5, "commuted")])
def test_sharded_solve_world4(tmp_path, oracle, case):
    """World size 4: uneven column / frequency splits (31 columns, 9 retained frequencies over 4
    ranks), the halo chain through three ranks."""
    _run_and_check(tmp_path, oracle, case, 4)


def _run_and_check(tmp_path, oracle, case, world):
    mp.spawn(_worker, args=(world, free_port(), case, str(tmp_path)), nprocs=world, join=True)
    parts = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    two_dim, g, n, nt, restart = case[:5]
    dt = 1.0 / nt
    if two_dim:
        po = oracle.problem_2d(g[0], g[1], 1.0, 1.0, 1.0 / (n + 1), n, nt, dt).build_plan()
        ns = n * n
    else:
        po = oracle.problem_1d(g[0], 1.0, 1.0 / (n + 1), n, nt, dt).build_plan()
        ns = n
    v = np.random.default_rng(5).uniform(-1, 1, nt * ns)
    cat = lambda key: np.concatenate([p[key] for p in parts])
    rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
    assert rel(cat("y"), po.matvec(v)) <= 1e-13
    assert rel(cat("z"), po.pc_apply(v)) <= 1e-11
    assert rel(cat("pf"), po.pc_forward(v)) <= 1e-11
    xo, ro = po.gmres(v, 1e-10, 200, restart=restart)
    assert all(int(p["iters"]) == ro.iterations for p in parts)
    assert rel(cat("x"), xo) <= 1e-10


def test_p2p_transport_needs_cuda_kernels():
    # the peer-store transport maps CUDA receive buffers: the numpy kernels are refused up front
    import pytest
    from paper_2003_07020_b200.distributed import ShardedSolver
    from dist_cpu_kernels import NumpyShardKernels
    with pytest.raises(ValueError):
        ShardedSolver(8, 7, NumpyShardKernels.__new__(NumpyShardKernels), transport="p2p")
    with pytest.raises(ValueError):
        ShardedSolver(8, 7, NumpyShardKernels.__new__(NumpyShardKernels), transport="mpi")
