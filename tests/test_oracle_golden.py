"""Pin the C oracle to the reference: the golden fixtures were produced by the reference itself
(tests/golden/make_golden.py over oracle/_ref), and, when oracle/_ref is present, live random
cases are compared too.  CPU only."""
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "fracpint_ref_golden.npz")
TAGS = ["p1a", "p1b", "p1c", "p1d", "p2a", "p2b", "p2c", "p1s", "p2s"]


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def make(oracle, prm):
    dim, g0, g1, k0, k1, h, n, nt, dt, alpha = prm
    if int(dim) == 1:
        p = oracle.problem_1d(g0, k0, h, int(n), int(nt), dt)
    else:
        p = oracle.problem_2d(g0, g1, k0, k1, h, int(n), int(nt), dt)
    return p.build_plan(alpha)


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def test_transforms_golden(oracle, gold):
    for n in (8, 12):
        x = gold[f"fft_in_{n}"]
        assert np.abs(oracle.fft(x, +1) - gold[f"fft_plus_{n}"]).max() <= 1e-13
        assert np.abs(oracle.fft(x, -1) - gold[f"fft_minus_{n}"]).max() <= 1e-13
    for n in (7, 10):
        assert np.abs(oracle.dst1(gold[f"dst_in_{n}"]) - gold[f"dst_out_{n}"]).max() <= 1e-14
        assert np.abs(oracle.dst1(gold[f"dstc_in_{n}"]) - gold[f"dstc_out_{n}"]).max() <= 1e-14
    for gamma in (1.2, 1.5, 1.8, 2.0):
        assert np.array_equal(oracle.centred_weights(gamma, 16), gold[f"weights_{gamma}"])
    assert np.abs(oracle.toeplitz_matvec(gold["toep_col"], gold["toep_v"]) - gold["toep_out"]).max() <= 1e-13
    assert np.abs(oracle.tau_spectrum(gold["tau_col"]) - gold["tau_sigma"]).max() <= 1e-13


@pytest.mark.parametrize("tag", TAGS)
def test_operator_plan_apply_golden(oracle, gold, tag):
    p = make(oracle, gold[f"{tag}_params"])
    v = gold[f"{tag}_v"]
    a, m = gold[f"{tag}_alpha_margin"]
    assert p.alpha == a
    assert abs(p.min_shift_margin - m) <= 1e-11 * m  # |lambda - dt sigma| min: cancellation
    assert np.abs(p.sigma() - gold[f"{tag}_sigma"]).max() <= 1e-13 * np.abs(gold[f"{tag}_sigma"]).max()
    assert rel(p.matvec(v), gold[f"{tag}_matvec"]) <= 1e-14
    # the alpha-scaled time FFTs amplify rounding: two faithful implementations differ by up to
    # ~1e-11 (oracle vs reference measured at config 0); 1e-11 is the pin for the PC apply
    assert rel(p.pc_apply(v, False), gold[f"{tag}_pc_half"]) <= 1e-11
    assert rel(p.pc_apply(v, True), gold[f"{tag}_pc_full"]) <= 1e-11
    assert rel(p.pc_forward(v), gold[f"{tag}_pc_forward"]) <= 1e-11


@pytest.mark.parametrize("tag", TAGS)
def test_gmres_golden(oracle, gold, tag):
    p = make(oracle, gold[f"{tag}_params"])
    x, rep = p.gmres(gold[f"{tag}_b"], 1e-10, 200)
    assert rep.iterations == int(gold[f"{tag}_iters"][0])
    assert rel(x, gold[f"{tag}_x"]) <= 1e-11
    assert np.abs(np.array(rep.residual_history) - gold[f"{tag}_history"]).max() <= 1e-12


@pytest.mark.parametrize("tag", TAGS)
def test_bicgstab_golden(oracle, gold, tag):
    """bicgstab_left (krylov.hpp:204-280): half-step iteration counts, x, history."""
    p = make(oracle, gold[f"{tag}_params"])
    x, rep = p.bicgstab(gold[f"{tag}_b"], 1e-10, 200)
    assert rep.iterations == float(gold[f"{tag}_bicg_iters"][0])
    assert rel(x, gold[f"{tag}_bicg_x"]) <= 1e-10
    h, g = np.array(rep.residual_history), gold[f"{tag}_bicg_history"]
    # late entries are norms of nearly cancelled residuals: compare them in units of ||b||
    assert len(h) == len(g) and np.allclose(h, g, rtol=1e-6, atol=1e-12)


def test_live_reference_pins(oracle, reference):
    """Random cases against the reference compiled here (skipped where oracle/_ref is absent)."""
    rng = np.random.default_rng(11)
    for gamma, ns, nt in [(1.3, 31, 8), (1.7, 63, 16), (1.5, 10, 5), (1.9, 127, 32)]:
        h, dt = 1.0 / (ns + 1), 1.0 / nt
        po = oracle.problem_1d(gamma, 1.0, h, ns, nt, dt).build_plan()
        pr = reference.problem_1d(gamma, 1.0, h, ns, nt, dt).build_plan()
        v = rng.uniform(-1, 1, ns * nt)
        assert rel(po.matvec(v), pr.matvec(v)) <= 1e-14
        assert rel(po.pc_apply(v), pr.pc_apply(v)) <= 1e-11
        if ns & (ns + 1) == 0 and nt & (nt - 1) == 0:
            # power-of-two transforms, both built with FMA contraction (oracle/Makefile): the
            # oracle's apply_inverse is the reference's to the bit
            assert np.array_equal(po.pc_apply(v), pr.pc_apply(v))
            assert np.array_equal(po.sigma(), pr.sigma())
        xo, ro = po.gmres(v, 1e-10, 200)
        xr, rr = pr.gmres(v, 1e-10, 200)
        assert ro.iterations == rr.iterations and rel(xo, xr) <= 1e-11
    po = oracle.problem_2d(1.3, 1.7, 1, 1, 1 / 8, 7, 8, 1 / 8).build_plan()
    pr = reference.problem_2d(1.3, 1.7, 1, 1, 1 / 8, 7, 8, 1 / 8).build_plan()
    v = rng.uniform(-1, 1, 49 * 8)
    assert rel(po.matvec(v), pr.matvec(v)) <= 1e-14 and rel(po.pc_apply(v), pr.pc_apply(v)) <= 1e-12


def test_live_reference_bicgstab(oracle, reference):
    rng = np.random.default_rng(12)
    for gamma, ns, nt, alpha in [(1.3, 31, 8, 0.0), (1.7, 63, 16, 1.0)]:
        h, dt = 1.0 / (ns + 1), 1.0 / nt
        po = oracle.problem_1d(gamma, 1.0, h, ns, nt, dt).build_plan(alpha)
        pr = reference.problem_1d(gamma, 1.0, h, ns, nt, dt).build_plan(alpha)
        b = rng.uniform(-1, 1, ns * nt)
        xo, ro = po.bicgstab(b, 1e-10, 200)
        xr, rr = pr.bicgstab(b, 1e-10, 200)
        assert ro.iterations == rr.iterations and rel(xo, xr) <= 1e-10
