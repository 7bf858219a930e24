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


def test_cpp_generic_gmres_and_plan_fields(tmp_path):
    """examples/plugin_gmres.cpp: the generic gmres_right(n, apply_a, apply_pinv, b, cfg) over host
    callables matches the device-resident solve; AlphaCirculantPlan carries the reference's
    scale_fwd / scale_bwd / tau fields; a callable's exception propagates."""
    if not shutil.which("g++"):
        pytest.skip("no g++")
    exe = str(tmp_path / "plugin_gmres")
    lib = os.path.join(ROOT, "paper_2003_07020_b200")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "plugin_gmres.cpp"), "-L" + lib, "-lfracpint_b200",
                    "-Wl,-rpath," + lib, "-o", exe], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    it_d, it_g, dx, trr, alpha, sf1, prod, sigma0, solve_count, taun, rethrown = out.stdout.split()
    assert abs(float(it_d) - float(it_g)) <= 1
    assert float(dx) <= 1e-10 and float(trr) <= 1e-9
    assert float(alpha) == 1.0 / 128  # min(0.5, dt/2), dt = 1/64
    assert abs(float(sf1) - (1.0 / 128) ** (1.0 / 64)) <= 1e-15 and abs(float(prod) - 1.0) <= 1e-15
    assert float(sigma0) < 0 and int(solve_count) == 33 and int(taun) == 255 and rethrown == "1"


def test_cpp_multi_device_example(tmp_path):
    """examples/multi_gpu_solve.cpp: the sharded solve through the C++ drop-in over 1, 2 and 4 ranks
    (all on device 0 on this box) equals the single-device solve."""
    if not shutil.which("g++"):
        pytest.skip("no g++")
    exe = str(tmp_path / "multi_gpu_solve")
    lib = os.path.join(ROOT, "paper_2003_07020_b200")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "multi_gpu_solve.cpp"), "-L" + lib, "-lfracpint_b200",
                    "-Wl,-rpath," + lib, "-o", exe], check=True)
    for devs in (["0"], ["0", "0"], ["0", "0", "0", "0"]):
        out = subprocess.run([exe, *devs], capture_output=True, text=True, timeout=120)
        assert out.returncode == 0, out.stdout + out.stderr
        ranks, it_s, it_1, dx, trr = out.stdout.split()
        assert int(ranks) == len(devs) and abs(float(it_s) - float(it_1)) <= 1
        assert float(dx) <= 1e-10 and float(trr) <= 1e-9
