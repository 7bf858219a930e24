"""Kernel variants selected by environment knobs agree with each other (each variant in its own
process: the knobs are read once):
  * time FFTs: the TMA-fed persistent kernels (kernels_time_tma.cu; n_time = 128..512 by default,
    1024 with FPC_TIME_TMA_1024=1) vs the register-staged column-tile / split kernels
    (FPC_TIME_TMA=0) -- the same arithmetic per element, so agreement to rounding;
  * the one-warp-per-transform kernels (n = 1023 lattice rows / columns, n_time = 1024 time FFTs) vs the
    CTA-level kernels they replaced (FPC_W32=0, FPC_TIME_WARP=0);
  * GMRES: the implicit re-orthogonalisation (stored basis never rewritten, host transformation
    matrix) vs the explicit U <- U - V a sweep (FPC_GS_IMPLICIT=0): same iteration count, same x."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def run_variant(tmp_path, name, env, cases):
    out = str(tmp_path / f"{name}.npz")
    r = subprocess.run([sys.executable, os.path.join(HERE, "variant_child.py"), out, *cases],
                       env={**os.environ, **env}, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    return np.load(out)


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def test_tma_time_ffts_match_register_staged(tmp_path):
    # ragged last tiles (n_space not a multiple of the tile width), odd and even n_space
    cases = ["pc:1d:8191:512", "pc:1d:8191:256", "pc:1d:16383:128", "pc:2d:127:256", "pc:2d:63:512"]
    a = run_variant(tmp_path, "tma", {"FPC_TIME_TMA": "1"}, cases)
    b = run_variant(tmp_path, "staged", {"FPC_TIME_TMA": "0"}, cases)
    for c in cases:
        assert rel(a[c], b[c]) <= 1e-13, (c, rel(a[c], b[c]))
        assert np.array_equal(a[c + ":mv"], b[c + ":mv"])  # the matvec does not depend on the knob


def test_tma_time_ffts_1024_match_split_kernels(tmp_path):
    cases = ["pc:1d:8191:1024", "pc:2d:127:1024"]
    # (the warp-owned n_time = 1024 kernels would take these sizes first: off in both variants)
    a = run_variant(tmp_path, "tma1k", {"FPC_TIME_TMA_1024": "1", "FPC_TIME_WARP": "0"}, cases)
    b = run_variant(tmp_path, "split", {"FPC_TIME_TMA_1024": "0", "FPC_TIME_WARP": "0"}, cases)
    for c in cases:
        assert rel(a[c], b[c]) <= 1e-13, (c, rel(a[c], b[c]))


def test_warp_time_ffts_1024_match_split_kernels(tmp_path):
    """kernels_time_warp.cu (one column per warp, the default from 2368 columns) vs the 2-CTA split
    kernels: odd and even n_space, a ragged last tile (8191 = 8 * 1023 + 7)."""
    cases = ["pc:1d:8191:1024", "pc:1d:4095:1024", "pc:2d:127:1024", "pc:2d:62:1024"]
    a = run_variant(tmp_path, "tw", {"FPC_TIME_WARP": "1"}, cases)
    b = run_variant(tmp_path, "split", {"FPC_TIME_WARP": "0"}, cases)
    for c in cases:
        assert rel(a[c], b[c]) <= 1e-13, (c, rel(a[c], b[c]))


def test_one_warp_per_transform_kernels_match_cta_kernels(tmp_path):
    """kernels_warp32.cu (n = 1023 rows / columns on 32 lanes x 32 registers) vs the CTA-level
    Stockham kernels (FPC_W32=0): matvec and PC apply in 2D and in 1D (2048 rows)."""
    cases = ["pc:2d:1023:4", "pc:1d:1023:2048"]
    a = run_variant(tmp_path, "w32", {"FPC_W32": "1"}, cases)
    b = run_variant(tmp_path, "cta", {"FPC_W32": "0"}, cases)
    for c in cases:
        # different factorisations of the transforms (32 x 32 / 16 x 32 against radix-16 Stockham
        # passes): rounding-level differences, amplified in the PC apply by the alpha^{-k/Nt}
        # scalings (1/alpha = 2 Nt) -- the tolerance of the PC apply against the oracle, 1e-12
        assert rel(a[c], b[c]) <= 1e-12, (c, rel(a[c], b[c]))
        assert rel(a[c + ":mv"], b[c + ":mv"]) <= 1e-14, (c, rel(a[c + ":mv"], b[c + ":mv"]))


def test_implicit_reorthogonalisation_matches_explicit(tmp_path):
    cases = ["solve:1d:1023:256", "solve:1d:4095:64", "solve:2d:63:64"]
    a = run_variant(tmp_path, "implicit", {"FPC_GS_IMPLICIT": "1"}, cases)
    b = run_variant(tmp_path, "explicit", {"FPC_GS_IMPLICIT": "0"}, cases)
    for c in cases:
        assert a[c + ":it"][0] == b[c + ":it"][0], (c, a[c + ":it"], b[c + ":it"])
        assert rel(a[c], b[c]) <= 1e-12, (c, rel(a[c], b[c]))
        assert a[c + ":it"][1] <= 1e-10 * 1.5
