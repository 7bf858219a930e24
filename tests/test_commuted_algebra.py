"""The commuted preconditioner ordering (kernels_commuted.cu) restated in numpy and
checked against the C oracle's reference-ordering apply (alpha_circulant.hpp:137-199) on CPU:
  P^{-1} v = (I (x) S) D^{-1} F^* diag[1/(lambda_n - dt sigma_i)] F D (I (x) S) v.
This pins the algebra the CUDA kernels implement; the GPU kernels are pinned in test_gpu_commuted.py."""
import numpy as np
import pytest


def dst_matrix(n):
    j = np.arange(1, n + 1)
    return np.sqrt(2.0 / (n + 1)) * np.sin(np.pi * np.outer(j, j) / (n + 1))


def commuted_apply(v, nt, ns, alpha, lam, sigma, dt, forward=False):
    S = dst_matrix(ns)
    V = v.reshape(nt, ns) @ S  # S symmetric: DST of every time level
    k = np.arange(nt)
    sf, sb = alpha ** (k / nt), alpha ** (-k / nt)
    Z = np.fft.ifft(sf[:, None] * V, axis=0) * nt  # e^{+2 pi i n k / Nt} (fft.hpp sign +1)
    d = lam[:, None] - dt * sigma[None, :]
    Y = Z * d if forward else Z / d
    U = (sb[:, None] * np.fft.fft(Y, axis=0) / nt).real
    return (U @ S).ravel()


@pytest.mark.parametrize("gamma,ns,nt,alpha", [(1.5, 15, 8, 0.0), (1.3, 31, 16, 0.0), (1.8, 7, 32, 1.0)])
def test_commuted_equals_reference_ordering(oracle, gamma, ns, nt, alpha):
    h, dt = 1.0 / (ns + 1), 1.0 / nt
    p = oracle.problem_1d(gamma, 1.0, h, ns, nt, dt).build_plan(alpha)
    v = np.random.default_rng(ns + nt).uniform(-1, 1, ns * nt)
    z = commuted_apply(v, nt, ns, p.alpha, p.lam(), p.sigma(), dt)
    zo = p.pc_apply(v)
    assert np.linalg.norm(z - zo) <= 1e-12 * np.linalg.norm(zo)
    zf = commuted_apply(v, nt, ns, p.alpha, p.lam(), p.sigma(), dt, forward=True)
    assert np.linalg.norm(zf - p.pc_forward(v)) <= 1e-12 * np.linalg.norm(zf)
