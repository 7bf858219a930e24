"""Dump PC applies (both orderings, half + full sweep, apply_forward) at config-1-like sizes with the
library FPC_LIB points at, for an A/B comparison of kernel variants: python split_check.py <tag>."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2003_07020_b200 as fp
from paper_2003_07020_b200 import problems

tag = sys.argv[1]
out = {}
for (gam, hinv, nt) in [(1.2, 8192, 2048), (1.5, 1024, 1024), (1.5, 512, 2048)]:
    w = problems.workload_1d(gam, hinv, nt)
    op = fp.AllAtOnceOperator(fp.TimeStencil(w.n_time), fp.RieszJacobian1D(gam, 1.0, w.h, w.n), w.dt)
    rng = np.random.default_rng(5)
    v = rng.standard_normal(w.n_time * w.n)
    for order in (fp.Ordering.reference, fp.Ordering.commuted):
        plan = fp.build_plan(fp.PreconditionerKind.generalized(), w.n_time, w.dt, op, ordering=order)
        out[f"{nt}_{w.n}_{order.name}_inv"] = fp.apply_inverse(plan, v)
        if order == fp.Ordering.reference:
            out[f"{nt}_{w.n}_{order.name}_full"] = fp.apply_inverse(plan, v, sweep=fp.InnerSweep.full)
        out[f"{nt}_{w.n}_{order.name}_fwd"] = fp.apply_forward(plan, v)
os.makedirs("gpurun_out", exist_ok=True)
np.savez(f"gpurun_out/split_{tag}.npz", **out)
if len(sys.argv) > 2:
    ref = np.load(f"gpurun_out/split_{sys.argv[2]}.npz")
    for k in out:
        a, b = out[k], ref[k]
        print(k, "rel diff %.3e" % (np.linalg.norm(a - b) / np.linalg.norm(b)))
