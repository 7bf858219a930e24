"""Achieved HBM bandwidth of the Gram-Schmidt vector kernels vs basis size (development aid).
Uses the shard entry points on config-1-sized vectors and the library's live kernel profile."""
import os, sys, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2003_07020_b200 as fp
from paper_2003_07020_b200 import _native as N

n = 8191 * 2048
ctx = fp.Context()
lib = N.load()
V = [torch.randn(n + 2, dtype=torch.float64, device="cuda") for _ in range(17)]
w = torch.randn(n + 2, dtype=torch.float64, device="cuda")
out = (C.c_double * 64)()
for nv in [1, 2, 4, 7, 8, 12, 16]:
    ptrs = (C.c_void_p * nv)(*[v.data_ptr() for v in V[:nv]])
    sc = (C.c_double * nv)(*([1e-3] * nv))
    for _ in range(2):
        N.check(lib.fpc_shard_dots(ctx.h, ptrs, sc, nv, C.c_void_p(w.data_ptr()), n, 1, out))
    with fp.KernelProfile() as pd:
        for _ in range(5):
            N.check(lib.fpc_shard_dots(ctx.h, ptrs, sc, nv, C.c_void_p(w.data_ptr()), n, 1, out))
    with fp.KernelProfile() as pu:
        for _ in range(5):
            N.check(lib.fpc_shard_update(ctx.h, ptrs, sc, nv, C.c_void_p(w.data_ptr()), n, out))
    ms_d = pd.table["dots"][0] / 5
    ms_u = pu.table["update"][0] / 5
    bd = (nv + 1) * n * 8 / ms_d / 1e6
    bu = (nv + 2) * n * 8 / ms_u / 1e6
    print(f"nv={nv:2d} dots {ms_d*1e3:7.1f} us {bd:7.0f} GB/s   update {ms_u*1e3:7.1f} us {bu:7.0f} GB/s")
