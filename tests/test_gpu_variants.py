"""Kernel variants selected by environment knobs agree with each other (each variant in its own
process: the knobs are read once):
  * time FFTs: the TMA-fed persistent kernels (kernels_time_tma.cu; n_time = 128..512 by default,
    1024 with FPC_TIME_TMA_1024=1) vs the register-staged column-tile / split kernels
    (FPC_TIME_TMA=0) -- the same arithmetic per element, so agreement to rounding;
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
    a = run_variant(tmp_path, "tma1k", {"FPC_TIME_TMA_1024": "1"}, cases)
    b = run_variant(tmp_path, "split", {"FPC_TIME_TMA_1024": "0"}, cases)
    for c in cases:
        assert rel(a[c], b[c]) <= 1e-13, (c, rel(a[c], b[c]))


def test_implicit_reorthogonalisation_matches_explicit(tmp_path):
    cases = ["solve:1d:1023:256", "solve:1d:4095:64", "solve:2d:63:64"]
    a = run_variant(tmp_path, "implicit", {"FPC_GS_IMPLICIT": "1"}, cases)
    b = run_variant(tmp_path, "explicit", {"FPC_GS_IMPLICIT": "0"}, cases)
    for c in cases:
        assert a[c + ":it"][0] == b[c + ":it"][0], (c, a[c + ":it"], b[c + ":it"])
        assert rel(a[c], b[c]) <= 1e-12, (c, rel(a[c], b[c]))
        assert a[c + ":it"][1] <= 1e-10 * 1.5
