"""Per-phase clock64 breakdown of the config-1 FFT kernels (development build with -DFPC_PHASE_TIMING,
scripts/_timing/libfpc_timing.so, scripts/build_timing.sh).  usage: phase_timing.py [mv|tau|time]"""
import os, sys, ctypes as C
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("FPC_LIB", os.path.join(ROOT, "scripts/_timing/libfpc_timing.so"))
import numpy as np, torch
import paper_2003_07020_b200 as fp
from paper_2003_07020_b200 import problems, _native as N

mode = sys.argv[1] if len(sys.argv) > 1 else "mv"
w = problems.config(1)
op = fp.AllAtOnceOperator(fp.TimeStencil(w.n_time), fp.RieszJacobian1D(w.gamma[0], 1.0, w.h, w.n), w.dt)
b = torch.from_numpy(problems.rhs(w)).cuda()
y = torch.empty_like(b)
if mode == "mv":
    run = lambda: (op.apply(b, y), op.ctx.synchronize())
    nb, sym = 2 * w.n_time, "fpc_debug_phases_mv"
    names = ["load(cp.async)+pretw", "fft_fwd", "pointwise", "fft_inv", "cluster_sync", "combine+stencil+store"]
elif mode == "time":
    plan = fp.build_plan(fp.PreconditionerKind.generalized(), w.n_time, w.dt, op)
    run = lambda: (fp.apply_inverse(plan, b, y), op.ctx.synchronize())
    for _ in range(3):
        run()
    lib = N.load()
    lib.fpc_debug_phases_t.argtypes = [C.c_void_p, C.c_int, C.c_int]
    nb = (w.n_space + 7) // 8
    for kid, nm in [(0, "time_fwd"), (1, "time_inv")]:
        buf = np.zeros((nb, 4), dtype=np.int64)
        assert lib.fpc_debug_phases_t(buf.ctypes.data, kid, nb) == 0
        d = np.diff(buf, axis=1)
        for i, n in enumerate(["load/pack", "fft", "unpack/store"]):
            print(f"{nm} {n:14s} mean {d[:, i].mean():9.0f} cyc  median {np.median(d[:, i]):9.0f}")
        print(f"{nm} per-CTA total mean {(buf[:, 3] - buf[:, 0]).mean():.0f}; CTAs {nb}")
    sys.exit(0)
else:
    plan = fp.build_plan(fp.PreconditionerKind.generalized(), w.n_time, w.dt, op)
    run = lambda: (fp.apply_inverse(plan, b, y), op.ctx.synchronize())
    nb, sym = w.n_time // 2 + 1, "fpc_debug_phases"
    names = ["load", "dst1", "divide", "dst2", "store"]
for _ in range(3):
    run()
op.ctx.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); run(); e1.record(); torch.cuda.synchronize()
print(mode, "ms", e0.elapsed_time(e1))
buf = np.zeros((nb, 16 if mode == "tau" else 8), dtype=np.int64)
lib = N.load()
getattr(lib, sym).argtypes = [C.c_void_p, C.c_int]
assert getattr(lib, sym)(buf.ctypes.data, nb) == 0
k = len(names)
d = np.diff(buf[:, :k + 1], axis=1)
for i, n in enumerate(names):
    print(f"{n:22s} mean {d[:, i].mean():9.0f} cyc  median {np.median(d[:, i]):9.0f}")
tot = buf[:, k] - buf[:, 0]
print("per-CTA total mean", tot.mean(), "cycles; CTAs", nb)
if mode == "tau":  # inside the second block_dst (stamps 8..11 are overwritten by the last call)
    dd = np.diff(buf[:, 8:12], axis=1)
    pre = buf[:, 8] - buf[:, 3]
    print(f"  dst2 pre            mean {pre.mean():9.0f}")
    for i, n in enumerate(["fft N", "fft N/2", "post"]):
        print(f"  dst2 {n:14s} mean {dd[:, i].mean():9.0f}")
