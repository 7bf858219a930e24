"""Build libfracpint_b200.so in-tree with nvcc for sm_100a (no torch JIT, no CPU fallback).

The shared library holds the CUDA kernels and the C-ABI (include/fracpint_b200.h); it is the
product.  `python -m paper_2003_07020_b200.build` or __graft_entry__.build() runs this.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
BUILD = os.path.join(ROOT, "build", "fpc")
LIB = os.path.join(HERE, "libfracpint_b200.so")
# "file.cu:N" compiles file.cu with -DFPC_1D_PART=N into file_pN.o (kernels_1d.cu is three units: its
# size instantiations took 3.5 of a cold build's 3.7 minutes in one nvcc process)
SOURCES = ["kernels_1d.cu:0", "kernels_1d.cu:1", "kernels_1d.cu:2", "kernels_mv.cu", "kernels_large.cu", "kernels_2d.cu", "kernels_full.cu",
           "kernels_krylov.cu", "kernels_commuted.cu", "kernels_tsplit.cu", "kernels_p2p.cu", "kernels_warp.cu", "kernels_warp32.cu", "kernels_generic.cu", "kernels_time_tma.cu", "kernels_time_warp.cu",
           "api.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# host code: x86-64-v3 with FMA contraction (g++'s C++ default once FMA exists), the arithmetic of the
# reference built with -march=native/-march=x86-64-v3: the host setup (weights, tau spectrum,
# circulant eigenvalues, lambda) is then bit-identical to the reference's (tests/test_abi.py)
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3,-march=x86-64-v3,-ffp-contract=fast",
         "--expt-relaxed-constexpr",
         "-diag-suppress", "39"]


def _stale(obj: str, deps: list[str]) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    stamp = os.path.join(BUILD, "flags.txt")
    flags = " ".join([NVCC, *ARCH, *FLAGS])
    if not os.path.exists(stamp) or open(stamp).read() != flags:
        force = True  # compiler flags changed: every object is stale
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers.append(os.path.join(ROOT, "include", "fracpint_b200.h"))
    jobs = []
    objs = []
    for spec in SOURCES:
        src, _, part = spec.partition(":")
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src.replace(".cu", f"_p{part}.o" if part else ".o"))
        objs.append(o)
        if force or _stale(o, [s] + headers):
            jobs.append([NVCC, *ARCH, *FLAGS, *([f"-DFPC_1D_PART={part}"] if part else []), "-c", s, "-o", o])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed: " + " ".join(cmd) + "\n" + r.stdout + r.stderr)
        return r.stdout + r.stderr

    with cf.ThreadPoolExecutor(max_workers=len(jobs) or 1) as ex:
        for out in ex.map(run, jobs):
            if verbose and out.strip():
                print(out)
    if force or jobs or not os.path.exists(LIB) or _stale(LIB, objs):
        run([NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-Xcompiler", "-fPIC"])
    with open(stamp, "w") as f:
        f.write(flags)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
