"""Device timings of matvec / PC apply at long spatial rows (config-4 upper range), development aid."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2003_07020_b200 as fp
from paper_2003_07020_b200 import problems

st = torch.cuda.Stream()
ctx = fp.Context(0, st)
for ns, nt in [(16383, 256), (32767, 256), (65535, 256)]:
    w = problems.workload_1d(1.5, ns + 1, nt)
    op = fp.AllAtOnceOperator(fp.TimeStencil(nt), fp.RieszJacobian1D(1.5, 1.0, w.h, w.n), w.dt, ctx)
    plan = fp.build_plan(fp.PreconditionerKind.generalized(), nt, w.dt, op)
    b = torch.randn(nt * ns, dtype=torch.float64, device="cuda")
    y = torch.empty_like(b)
    def t(fn, reps=20):
        with torch.cuda.stream(st):
            for _ in range(3): fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(reps): fn()
            e1.record(st)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps * 1e3
    tm, tp = t(lambda: op.apply(b, y)), t(lambda: fp.apply_inverse(plan, b, y))
    N = ns * nt
    print(f"ns {ns} nt {nt}: matvec {tm:.1f} us ({16 * N / tm / 1e3:.0f} GB/s)  pc {tp:.1f} us ({(16 * N + 64 * (nt // 2 + 1) * ns) / tp / 1e3:.0f} GB/s)")
