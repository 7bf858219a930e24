import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2003_07020_b200 as fp
ns, nt = int(sys.argv[1]), int(sys.argv[2])
op = fp.AllAtOnceOperator(fp.TimeStencil(nt), fp.RieszJacobian1D(1.5, 1.0, 1/(ns+1), ns), 1/nt)
plan = fp.build_plan(fp.PreconditionerKind.generalized(), nt, 1/nt, op)
v = np.random.default_rng(0).uniform(-1, 1, ns*nt)
try:
    z = fp.apply_inverse(plan, v)
    print("ok", ns, nt)
except Exception as e:
    print("FAIL", ns, nt, e)
