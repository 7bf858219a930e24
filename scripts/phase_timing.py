"""Per-phase clock64 breakdown of k_matvec_1d_split (build/timing/libfpc_timing.so, -DFPC_PHASE_TIMING)."""
import os, sys, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("FPC_LIB", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "build/timing/libfpc_timing.so"))
import numpy as np, torch
import paper_2003_07020_b200 as fp
from paper_2003_07020_b200 import problems, _native as N
w = problems.config(1)
op = fp.AllAtOnceOperator(fp.TimeStencil(w.n_time), fp.RieszJacobian1D(w.gamma[0], 1.0, w.h, w.n), w.dt)
b = torch.from_numpy(problems.rhs(w)).cuda()
y = torch.empty_like(b)
for _ in range(3): op.apply(b, y)
op.ctx.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); op.apply(b, y); e1.record(); torch.cuda.synchronize()
print("kernel ms", e0.elapsed_time(e1))
nb = 2 * w.n_time
buf = np.zeros((nb, 8), dtype=np.int64)
lib = N.load()
lib.fpc_debug_phases_mv.argtypes = [C.c_void_p, C.c_int]
assert lib.fpc_debug_phases_mv(buf.ctypes.data, nb) == 0
names = ["load(cp.async)+pretw", "fft_fwd", "pointwise", "fft_inv", "cluster_sync", "combine+stencil+store"]
d = np.diff(buf[:, :7], axis=1)
for i, n in enumerate(names):
    print(f"{n:22s} mean {d[:, i].mean():9.0f} cyc  median {np.median(d[:, i]):9.0f}")
tot = buf[:, 6] - buf[:, 0]
print("per-CTA total mean", tot.mean(), "cycles; CTAs", nb)
span = buf[:, 6].max() - buf[:, 0].min()
print("span (cycles, across SMs clocks may differ)", span)
