"""The C++ drop-in header (include/fracpint_b200.hpp) compiled against libfracpint_b200.so and run:
the reference's library-usage sequence (proj/README.md 'Library usage') with GPU underneath."""
import os
import shutil
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_dropin_example(tmp_path):
    if not shutil.which("g++"):
        pytest.skip("no g++")
    exe = str(tmp_path / "dropin_solve")
    lib = os.path.join(ROOT, "paper_2003_07020_b200")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "dropin_solve.cpp"), "-L" + lib, "-lfracpint_b200",
                    "-Wl,-rpath," + lib, "-o", exe], check=True)
    out = subprocess.run([exe, "256", "64"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    ns, nt, iters, trr, trr_host, _ = out.stdout.split()
    assert (int(ns), int(nt)) == (255, 64)
    assert 1 <= float(iters) <= 20
    assert float(trr) <= 1e-9
    assert abs(float(trr_host) - float(trr)) <= 1e-3 * float(trr) + 1e-15
