"""Per-operator device times of a BASELINE config on the library stream (development aid for A/B
runs: e.g. FPC_WARP=0 python scripts/kernel_ab.py 2).  Prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2003_07020_b200 as fp  # noqa: E402
from paper_2003_07020_b200 import problems  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
w = problems.config(cfg)
stream = torch.cuda.Stream()
ctx = fp.Context(0, stream)
jac = (fp.RieszJacobian2D(w.gamma[0], w.gamma[1], 1.0, 1.0, w.h, w.n) if w.two_dim
       else fp.RieszJacobian1D(w.gamma[0], 1.0, w.h, w.n))
op = fp.AllAtOnceOperator(fp.TimeStencil(w.n_time), jac, w.dt, ctx)
plan = fp.build_plan(fp.PreconditionerKind.generalized(), w.n_time, w.dt, op)
with torch.cuda.stream(stream):
    b = torch.from_numpy(problems.rhs(w)).cuda()
    y = torch.empty_like(b)
stream.synchronize()
out = {"config": w.name, "FPC_WARP": os.environ.get("FPC_WARP", "1")}
for name, fn in (("matvec", lambda: op.apply(b, y)), ("pc", lambda: fp.apply_inverse(plan, b, y))):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    with fp.KernelProfile() as prof:
        for _ in range(reps):
            fn()
    out[name + "_ms"] = e0.elapsed_time(e1) / reps
    out[name + "_kernels_us"] = {k: round(1e3 * v[0] / v[1], 1) for k, v in prof.table.items()}
print(json.dumps(out))
