"""Device-resident solve time of BASELINE configs (CUDA events on the library stream; development
aid for A/B runs).  Usage: python scripts/solve_timing.py 0 2 [reps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2003_07020_b200 as fp  # noqa: E402
from paper_2003_07020_b200 import problems  # noqa: E402

reps = 20
cfgs = [int(a) for a in sys.argv[1:] if a.isdigit() and int(a) <= 3] or [0]
for c in cfgs:
    w = problems.config(c)
    stream = torch.cuda.Stream()
    ctx = fp.Context(0, stream)
    jac = (fp.RieszJacobian2D(w.gamma[0], w.gamma[1], 1.0, 1.0, w.h, w.n) if w.two_dim
           else fp.RieszJacobian1D(w.gamma[0], 1.0, w.h, w.n))
    op = fp.AllAtOnceOperator(fp.TimeStencil(w.n_time), jac, w.dt, ctx)
    order = fp.Ordering.commuted if "commuted" in sys.argv else fp.Ordering.reference
    plan = fp.build_plan(fp.PreconditionerKind.generalized(), w.n_time, w.dt, op, ordering=order)
    cfg = fp.SolverConfig(tol=w.tol, max_iter=200, restart=w.restart)
    with torch.cuda.stream(stream):
        b = torch.from_numpy(problems.rhs(w)).cuda()
        x = torch.empty_like(b)
    stream.synchronize()
    for _ in range(3):
        r = fp.gmres_right(op, plan, b, cfg, out=x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        r = fp.gmres_right(op, plan, b, cfg, out=x)
    e1.record(stream)
    torch.cuda.synchronize()
    with fp.KernelProfile() as prof:
        fp.gmres_right(op, plan, b, cfg, out=x)
    print(json.dumps({"config": w.name, "ms": e0.elapsed_time(e1) / reps, "iterations": r.report.iterations,
                      "trr": r.report.true_relative_residual,
                      "kernels_ms": {k: round(v[0], 4) for k, v in prof.table.items()}}))
