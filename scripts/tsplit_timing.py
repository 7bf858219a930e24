"""PC apply timings (both orderings) at long time series, development aid for the time-split kernels."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2003_07020_b200 as fp
from paper_2003_07020_b200 import problems

st = torch.cuda.Stream()
ctx = fp.Context(0, st)
for ns, nt in [(8191, 2048), (1023, 4096), (8191, 4096), (1023, 8192), (4095, 8192)]:
    w = problems.workload_1d(1.5, ns + 1, nt)
    op = fp.AllAtOnceOperator(fp.TimeStencil(nt), fp.RieszJacobian1D(1.5, 1.0, w.h, w.n), w.dt, ctx)
    b = torch.randn(nt * ns, dtype=torch.float64, device="cuda")
    y = torch.empty_like(b)
    out = []
    for order in (fp.Ordering.reference, fp.Ordering.commuted):
        plan = fp.build_plan(fp.PreconditionerKind.generalized(), nt, w.dt, op, ordering=order)
        with torch.cuda.stream(st):
            for _ in range(3): fp.apply_inverse(plan, b, y)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(10): fp.apply_inverse(plan, b, y)
            e1.record(st)
            with fp.KernelProfile() as prof:
                fp.apply_inverse(plan, b, y)
        torch.cuda.synchronize()
        out.append(f"{order.name} {e0.elapsed_time(e1) / 10 * 1e3:.1f} us " + str({k: round(v[0] / v[1] * 1e3, 1) for k, v in prof.table.items()}))
    print(f"ns {ns} nt {nt}: " + " | ".join(out))
