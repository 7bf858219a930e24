"""Known-answer and dense-oracle checks of the C oracle, restated (Eigen-free) from the reference's
own Catch2 suites.  Each test cites the reference test it restates.  CPU only."""
import math

import numpy as np
import pytest

from oracle.oracle import OracleError, OracleInvalidArgument


def dst_matrix(n):
    i = np.arange(1, n + 1)
    return np.sqrt(2.0 / (n + 1)) * np.sin(np.pi * np.outer(i, i) / (n + 1))


def dense_toeplitz(col):
    n = len(col)
    return np.array([[col[abs(i - j)] for j in range(n)] for i in range(n)])


# ---- transforms (test_transforms.cpp) --------------------------------------------------------
def test_dft_sign_kat(oracle):
    # test_transforms.cpp:23-39: forward unitary DFT of e_2 (0-based e_1) is 1/2 [1, i, -1, -i]
    x = np.zeros(4, complex)
    x[1] = 1.0
    y = oracle.fft(x, +1) / 2.0
    assert np.allclose(y, 0.5 * np.array([1, 1j, -1, -1j]), atol=1e-15)


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 12, 100, 1024, 4096])
def test_dft_roundtrip_and_naive(oracle, n):
    # test_transforms.cpp:41-67: inverse undoes forward, and agrees with the quadratic-time DFT
    rng = np.random.default_rng(n)
    x = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
    y = oracle.fft(x, +1)
    back = oracle.fft(y, -1) / n
    assert np.abs(back - x).max() <= 1e-12 * (1 + np.linalg.norm(x))
    if n <= 128:
        k = np.arange(n)
        naive = np.exp(2j * np.pi * np.outer(k, k) / n) @ x
        assert np.abs(y - naive).max() <= 1e-10 * (1 + np.linalg.norm(x))


def test_dst_trivial_sizes(oracle):
    # test_transforms.cpp:78-88: n = 1 is the identity; n = 2 maps [1, 0] to [1/sqrt2, 1/sqrt2]
    assert np.allclose(oracle.dst1(np.array([3.0])), [3.0], atol=1e-15)
    assert np.allclose(oracle.dst1(np.array([1.0, 0.0])), [2 ** -0.5, 2 ** -0.5], atol=1e-15)


@pytest.mark.parametrize("n", [1, 3, 7, 10, 31, 64])
def test_dst_oracle_involution_complex(oracle, n):
    # test_transforms.cpp:90-122: matches the dense DST matrix, is involutory, complex = componentwise
    rng = np.random.default_rng(n)
    x = rng.uniform(-1, 1, n)
    z = x + 1j * rng.uniform(-1, 1, n)
    Q = dst_matrix(n)
    assert np.abs(oracle.dst1(x) - Q @ x).max() <= 1e-12
    assert np.abs(oracle.dst1(oracle.dst1(x)) - x).max() <= 1e-12
    assert np.abs(oracle.dst1(z) - (oracle.dst1(z.real) + 1j * oracle.dst1(z.imag))).max() <= 1e-13


def test_toeplitz_pinned(oracle):
    # test_transforms.cpp:124-135
    v = np.array([4.0, -3.0, 2.0, -1.0])
    assert np.abs(oracle.toeplitz_matvec([1.0, 0, 0, 0], v) - v).max() <= 1e-13
    out = oracle.toeplitz_matvec([2.0, -1.0, 0, 0, 0], np.arange(1.0, 6.0))
    assert np.abs(out - [0, 0, 0, 0, 6.0]).max() <= 1e-12


def test_toeplitz_random_dense(oracle):
    # test_transforms.cpp:137-161 (100 random instances)
    rng = np.random.default_rng(20260819)
    for _ in range(100):
        n = 1 + int(rng.uniform(0, 127.99))
        col, v = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
        ref = dense_toeplitz(col) @ v
        assert np.abs(oracle.toeplitz_matvec(col, v) - ref).max() <= 1e-12 * (1 + np.linalg.norm(ref))


def test_tau_spectrum_kats(oracle):
    # test_transforms.cpp:163-184: identity -> 1; Laplacian -> 2 - 2cos(pi i/(n+1)); frozen n = 3
    assert np.allclose(oracle.tau_spectrum([1.0, 0, 0, 0, 0, 0]), 1.0, atol=1e-13)
    for n in (1, 3, 7, 16):
        col = np.zeros(n)
        col[0] = 2.0
        if n > 1:
            col[1] = -1.0
        i = np.arange(1, n + 1)
        assert np.abs(oracle.tau_spectrum(col) - (2 - 2 * np.cos(np.pi * i / (n + 1)))).max() <= 1e-12
    s3 = oracle.tau_spectrum([2.0, -1.0, 0.0])
    assert np.abs(s3 - [0.5857864376269049, 2.0, 3.414213562373095]).max() <= 1e-13


def test_tau_is_hankel_corrected_toeplitz(oracle):
    # test_transforms.cpp:186-212: tau(T) = T - H, H(i,j) = a[i+j+2] + a[2n-i-j] (0-based)
    rng = np.random.default_rng(3)
    n = 9
    a = rng.uniform(-1, 1, n)
    Q = dst_matrix(n)
    tau = Q @ np.diag(oracle.tau_spectrum(a)) @ Q
    ext = np.r_[a, np.zeros(n + 3)]
    H = np.array([[ext[i + j + 2] + (ext[2 * n - i - j] if 2 * n - i - j < len(ext) else 0.0)
                   for j in range(n)] for i in range(n)])
    assert np.abs(tau - (dense_toeplitz(a) - H)).max() <= 1e-12


def test_tau_solve_shifted_vs_dense_and_singular(oracle):
    # test_transforms.cpp:214-248
    rng = np.random.default_rng(4)
    n = 12
    sigma = -rng.uniform(0.5, 5.0, n)
    shift, dt = 1.5 - 0.3j, 0.1
    rhs = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
    Q = dst_matrix(n)
    dense = shift * np.eye(n) - dt * (Q @ np.diag(sigma) @ Q)
    out = oracle.tau_solve_shifted(sigma, 0, 0, shift, dt, rhs)
    assert np.abs(out - np.linalg.solve(dense, rhs)).max() <= 1e-12
    with pytest.raises(OracleError):
        oracle.tau_solve_shifted(np.ones(4), 0, 0, 0.1 + 0j, 0.1, np.ones(4, complex))


# ---- discretisation (test_discretization.cpp) ------------------------------------------------
def test_weights_kats(oracle):
    # :31-42 gamma = 2 gives [2, -1, 0...]; gamma = 1.5 frozen values
    w2 = oracle.centred_weights(2.0, 6)
    assert abs(w2[0] - 2.0) <= 1e-14 and abs(w2[1] + 1.0) <= 1e-14 and np.abs(w2[2:]).max() <= 1e-14
    w = oracle.centred_weights(1.5, 3)
    assert w[0] == pytest.approx(1.573787, rel=1e-5) and w[1] == pytest.approx(-0.674480, rel=1e-5)


@pytest.mark.parametrize("gamma", [1.1, 1.3, 1.5, 1.7, 1.9, 1.99])
def test_weights_reflected_gamma(oracle, gamma):
    # :19-23, 44-54: w_l = -sin(pi g/2)/pi * exp(lgamma(1+g) + lgamma(l-g/2) - lgamma(1+g/2+l))
    w = oracle.centred_weights(gamma, 65)
    for l in range(1, 65):
        ref = -math.sin(math.pi * gamma / 2) / math.pi * math.exp(
            math.lgamma(1 + gamma) + math.lgamma(l - gamma / 2) - math.lgamma(1 + gamma / 2 + l))
        assert w[l] == pytest.approx(ref, rel=1e-12, abs=1e-300)


def test_weights_reject(oracle):
    with pytest.raises(OracleInvalidArgument):
        oracle.centred_weights(0.5, 4)
    with pytest.raises(OracleInvalidArgument):
        oracle.centred_weights(1.5, 0)


def test_jacobian_frozen_column(oracle):
    # :89-99
    lap = oracle.problem_1d(2.0, 1.0, 1.0, 3, 4, 0.1)
    c = lap.column()
    assert abs(c[0] + 2) <= 1e-13 and abs(c[1] - 1) <= 1e-13 and abs(c[2]) <= 1e-13
    frac = oracle.problem_1d(1.5, 0.01, 1.0 / 128.0, 8, 4, 0.1)
    c = frac.column()
    assert c[0] == pytest.approx(-22.7909, rel=1e-4)
    assert np.all(c[1:] > 0)


# ---- all-at-once operator (test_allatonce.cpp) -------------------------------------------------
def dense_op(p):
    N = p.n
    A = np.zeros((N, N))
    e = np.zeros(N)
    for j in range(N):
        e[j] = 1.0
        A[:, j] = p.matvec(e)
        e[j] = 0.0
    return A


def test_matvec_dense_kron(oracle):
    # test_allatonce.cpp:113-134: C (x) I - dt I (x) A
    nt, ns, dt = 5, 6, 0.2
    p = oracle.problem_1d(1.6, 0.3, 1.0 / 7, ns, nt, dt)
    col = p.column()
    A = dense_toeplitz(col)
    C = np.zeros((nt, nt))
    C[0, 0] = 1.0
    for k in range(1, nt):
        C[k, k], C[k, k - 1] = 1.5, -2.0
        if k >= 2:
            C[k, k - 2] = 0.5
    ref = np.kron(C, np.eye(ns)) - dt * np.kron(np.eye(nt), A)
    assert np.abs(dense_op(p) - ref).max() <= 1e-12 * np.abs(ref).max()


def test_rhs_assembly(oracle):
    # test_allatonce.cpp:136-158
    nt, ns, dt = 4, 3, 0.25
    f = np.arange(nt * ns, dtype=float)
    u0 = np.array([1.0, 2.0, 3.0])
    b = oracle.assemble_rhs(nt, ns, dt, f, u0)
    ref = dt * f
    ref[:ns] += u0
    ref[ns:2 * ns] -= 0.5 * u0
    assert np.array_equal(b, ref)


# ---- preconditioner (test_pint.cpp) ------------------------------------------------------------
def test_alpha_policy_and_eigenvalues(oracle):
    # :59-92: alpha_for(0.004) = 0.002; Strang lambda_0 = 0, Re = (1 - cos)^2; conjugate pairs
    p = oracle.problem_1d(1.5, 1.0, 0.25, 3, 4, 0.004).build_plan()
    assert p.alpha == pytest.approx(0.002)
    for nt in (4, 16, 64, 1024):
        lam = oracle.alpha_circulant_eigenvalues(1.0, nt)
        assert abs(lam[0]) <= 1e-13
        c = np.cos(2 * np.pi * np.arange(nt) / nt)
        assert np.abs(lam.real - (1 - c) ** 2).max() <= 1e-12
    for alpha in (0.01, 0.1, 0.5, 0.9):
        lam = oracle.alpha_circulant_eigenvalues(alpha, 64)
        assert np.all(lam.real > 0)
        assert np.abs(lam[1:][::-1] - np.conj(lam[1:])).max() <= 1e-13


def dense_precond(p, alpha, nt, ns, dt, sigma, nx=0):
    r = [1.5, -2.0, 0.5]
    C = np.zeros((nt, nt))
    for i in range(nt):
        for j in range(nt):
            d = i - j
            if 0 <= d <= 2:
                C[i, j] = r[d]
            if d < 0 and d + nt <= 2:
                C[i, j] = alpha * r[d + nt]
    if nx:
        Q = np.kron(dst_matrix(nx), dst_matrix(nx))
    else:
        Q = dst_matrix(ns)
    tau = Q @ np.diag(sigma) @ Q
    return np.kron(C, np.eye(ns)) - dt * np.kron(np.eye(nt), tau)


@pytest.mark.parametrize("nt", [4, 5])
@pytest.mark.parametrize("alpha", [0.5, 1.0])
def test_apply_inverse_dense_lu(oracle, nt, alpha):
    # :149-171 (1D), both sweeps
    ns = 4
    p = oracle.problem_1d(1.5, 0.02, 1.0 / (ns + 1), ns, nt, 0.25).build_plan(alpha)
    P = dense_precond(p, alpha, nt, ns, 0.25, p.sigma())
    v = np.random.default_rng(nt).uniform(-1, 1, nt * ns)
    ref = np.linalg.solve(P, v)
    for full in (False, True):
        assert np.abs(p.pc_apply(v, full) - ref).max() <= 1e-10 * (1 + np.linalg.norm(ref))


def test_apply_inverse_dense_lu_2d(oracle):
    # :173-186
    nt, n = 5, 3
    p = oracle.problem_2d(1.4, 1.8, 0.03, 0.05, 0.25, n, nt, 0.2).build_plan(0.6)
    P = dense_precond(p, 0.6, nt, n * n, 0.2, p.sigma(), nx=n)
    v = np.random.default_rng(1).uniform(-1, 1, nt * n * n)
    ref = np.linalg.solve(P, v)
    assert np.abs(p.pc_apply(v) - ref).max() <= 1e-10 * (1 + np.linalg.norm(ref))


def test_forward_roundtrip_and_half_full(oracle):
    # :188-216
    p = oracle.problem_1d(1.9, 0.4, 0.2, 6, 6, 0.15).build_plan(0.35)
    v = np.random.default_rng(2).uniform(-1, 1, 36)
    assert np.abs(p.pc_apply(p.pc_forward(v)) - v).max() <= 1e-10 * (1 + np.linalg.norm(v))
    for nt in (4, 5, 6, 7, 16):
        q = oracle.problem_1d(1.7, 0.05, 1.0 / 7, 6, nt, 1.0 / nt).build_plan()
        w = np.random.default_rng(nt).uniform(-1, 1, nt * 6)
        full = q.pc_apply(w, True)
        assert np.abs(q.pc_apply(w, False) - full).max() <= 1e-12 * (1 + np.linalg.norm(full))


def test_singular_plan_rejected(oracle):
    # test_pint.cpp:140-147 uses ZeroJacobian + Strang; here lambda_0 = 0 with alpha = 1 and a tiny
    # spatial operator is not exactly singular, so check the alpha range guard instead
    p = oracle.problem_1d(1.5, 1.0, 0.25, 3, 8, 0.1)
    with pytest.raises(OracleInvalidArgument):
        p.build_plan(1.5)


# ---- Krylov (test_krylov.cpp) ----------------------------------------------------------------
def test_gmres_matches_dense_solve(oracle):
    # test_krylov.cpp:150-185
    nt, ns, dt = 6, 5, 0.2
    p = oracle.problem_1d(1.5, 0.02, 1.0 / (ns + 1), ns, nt, dt).build_plan()
    b = np.random.default_rng(7).uniform(-1, 1, nt * ns)
    ref = np.linalg.solve(dense_op(p), b)
    x, rep = p.gmres(b, 1e-9, 200)
    assert rep.converged and rep.iterations <= 10
    assert np.abs(x - ref).max() <= 1e-7 * (1 + np.linalg.norm(ref))
    hist = np.array(rep.residual_history)
    assert np.all(np.diff(hist) <= 1e-15)  # test_krylov.cpp:63-73 monotone history


def test_gmres_zero_rhs_and_budget(oracle):
    # test_krylov.cpp:126-148
    p = oracle.problem_1d(1.5, 1.0, 1.0 / 16, 15, 8, 0.125).build_plan()
    x, rep = p.gmres(np.zeros(15 * 8), 1e-9, 200)
    assert rep.converged and rep.iterations == 0 and not np.any(x)
    x, rep = p.gmres(np.random.default_rng(0).uniform(-1, 1, 120), 1e-15, 3)
    assert not rep.converged and rep.iterations == 3 and len(rep.residual_history) == 3


def test_restart_emulation_converges(oracle):
    # GMRES(m) built on the unrestarted routine
    p = oracle.problem_1d(1.5, 1.0, 1.0 / 64, 63, 16, 1.0 / 16).build_plan()
    b = np.random.default_rng(1).uniform(-1, 1, 63 * 16)
    x_full, r_full = p.gmres(b, 1e-10, 200)
    for m in (3, 5, 20):
        x, rep = p.gmres(b, 1e-10, 200, restart=m)
        assert rep.converged
        assert np.linalg.norm(x - x_full) <= 1e-8 * np.linalg.norm(x_full)
        assert rep.true_relative_residual <= 1e-9
