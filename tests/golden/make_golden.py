"""Generate tests/golden/fracpint_ref_golden.npz from the REFERENCE itself.

The reference (/root/reference/proj/include/fracpint, header-only C++20) is compiled unchanged into
oracle/_ref/libfracpint_ref.so by oracle/Makefile (ref_shim.cpp only calls its public API).  This
script drives it on small seeded cases and stores inputs and outputs; the fixtures pin both the C
oracle (tests/test_oracle_golden.py) and the GPU path (tests/test_gpu_golden.py) on machines
without /root/reference.  Re-run: `make -C oracle && python tests/golden/make_golden.py`.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import Reference  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "fracpint_ref_golden.npz")


def main():
    r = Reference()
    r.set_threads(1)
    rng = np.random.default_rng(20260819)
    g = {}
    # transforms (fft.hpp, dst.hpp): power-of-two and Bluestein sizes
    for n in (8, 12):
        x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        g[f"fft_in_{n}"] = x
        g[f"fft_plus_{n}"] = r.fft(x, +1)
        g[f"fft_minus_{n}"] = r.fft(x, -1)
    for n in (7, 10):
        x = rng.standard_normal(n)
        z = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        g[f"dst_in_{n}"], g[f"dst_out_{n}"] = x, r.dst1(x)
        g[f"dstc_in_{n}"], g[f"dstc_out_{n}"] = z, r.dst1(z)
    # weights.hpp
    for gamma in (1.2, 1.5, 1.8, 2.0):
        g[f"weights_{gamma}"] = r.centred_weights(gamma, 16)
    # toeplitz.hpp / tau.hpp
    col = rng.uniform(-1, 1, 20)
    v = rng.uniform(-1, 1, 20)
    g["toep_col"], g["toep_v"], g["toep_out"] = col, v, r.toeplitz_matvec(col, v)
    col = -np.abs(rng.uniform(0.5, 1.0, 15)) * np.r_[-2.0, np.ones(14)]
    g["tau_col"], g["tau_sigma"] = col, r.tau_spectrum(col)
    # operator / plan / apply / GMRES cases: (tag, dim, gammas, kappas, h, n, nt, dt, alpha)
    cases = [
        ("p1a", 1, (1.5,), (1.0,), 1.0 / 16, 15, 8, 1.0 / 8, 0.0),
        ("p1b", 1, (1.2,), (0.5,), 1.0 / 64, 63, 16, 1.0 / 16, 0.0),
        ("p1c", 1, (1.8,), (1.0,), 1.0 / 32, 31, 32, 1.0 / 32, 0.25),
        ("p1d", 1, (1.5,), (1.0,), 1.0 / 128, 127, 32, 1.0 / 32, 0.0),
        ("p2a", 2, (1.3, 1.7), (1.0, 1.0), 1.0 / 8, 7, 8, 1.0 / 8, 0.0),
        ("p2b", 2, (1.4, 1.8), (0.03, 0.05), 0.25, 7, 8, 0.2, 0.6),
        ("p2c", 2, (1.5, 1.5), (1.0, 1.0), 1.0 / 16, 15, 16, 1.0 / 16, 0.0),
        # Strang P1 (alpha = 1, lambda_0 = 0; alpha_circulant.hpp:26)
        ("p1s", 1, (1.5,), (1.0,), 1.0 / 32, 31, 16, 1.0 / 16, 1.0),
        ("p2s", 2, (1.3, 1.7), (1.0, 1.0), 1.0 / 8, 7, 8, 1.0 / 8, 1.0),
    ]
    for tag, dim, gm, kp, h, n, nt, dt, alpha in cases:
        if dim == 1:
            p = r.problem_1d(gm[0], kp[0], h, n, nt, dt)
            ns = n
        else:
            p = r.problem_2d(gm[0], gm[1], kp[0], kp[1], h, n, nt, dt)
            ns = n * n
        p.build_plan(alpha)
        N = ns * nt
        v = rng.uniform(-1, 1, N)
        b = rng.uniform(-1, 1, N)
        x, rep = p.gmres(b, 1e-10, 200)
        g[f"{tag}_params"] = np.array([dim, gm[0], gm[-1], kp[0], kp[-1], h, n, nt, dt, alpha])
        g[f"{tag}_v"] = v
        g[f"{tag}_matvec"] = p.matvec(v)
        g[f"{tag}_pc_half"] = p.pc_apply(v, False)
        g[f"{tag}_pc_full"] = p.pc_apply(v, True)
        g[f"{tag}_pc_forward"] = p.pc_forward(v)
        g[f"{tag}_sigma"] = p.sigma()
        g[f"{tag}_alpha_margin"] = np.array([p.alpha, p.min_shift_margin])
        g[f"{tag}_b"] = b
        g[f"{tag}_x"] = x
        g[f"{tag}_iters"] = np.array([rep.iterations])
        g[f"{tag}_history"] = np.array(rep.residual_history)
        g[f"{tag}_trr"] = np.array([rep.true_relative_residual])
        # bicgstab_left (krylov.hpp:204-280) on the same system
        xb, rb = p.bicgstab(b, 1e-10, 200)
        g[f"{tag}_bicg_x"] = xb
        g[f"{tag}_bicg_iters"] = np.array([rb.iterations])
        g[f"{tag}_bicg_history"] = np.array(rb.residual_history)
        g[f"{tag}_bicg_trr"] = np.array([rb.true_relative_residual])
    # paper-table path: run_problem on the manufactured benchmarks (driver.hpp:94-112).
    # (tag, dim, gx, gy, nt, h_inv, method, strang, keep_rhs)
    rows = [
        ("rp1a", 1, 1.2, 0.0, 64, 128, "gmres", False, True),
        ("rp1b", 1, 1.2, 0.0, 64, 128, "gmres", True, False),
        ("rp1c", 1, 1.9, 0.0, 64, 128, "gmres", False, False),
        ("rp1d", 1, 1.5, 0.0, 16, 32, "bicgstab", False, True),
        ("rp2a", 2, 1.4, 1.2, 16, 16, "bicgstab", False, True),
        ("rp2b", 2, 1.5, 1.5, 64, 64, "bicgstab", False, False),
        ("rp2c", 2, 1.5, 1.5, 64, 64, "bicgstab", True, False),
        ("rp2d", 2, 1.7, 1.9, 16, 16, "gmres", False, False),
    ]
    for tag, dim, gx, gy, nt, h_inv, method, strang, keep in rows:
        out = r.run_problem(dim, gx, gy, nt, h_inv, method, strang)
        g[f"{tag}_params"] = np.array([dim, gx, gy, nt, h_inv, 1 if method == "bicgstab" else 0, int(strang)])
        g[f"{tag}_result"] = np.array([out["iterations"], float(out["converged"]), out["err_inf"]])
        g[f"{tag}_final"] = out["final"]
        g[f"{tag}_exact"] = out["exact"]
        if keep:
            g[f"{tag}_rhs"] = out["rhs"]
    np.savez_compressed(OUT, **g)
    print("wrote", OUT, os.path.getsize(OUT), "bytes,", len(g), "arrays")


if __name__ == "__main__":
    main()
