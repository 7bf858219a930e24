"""n_time = 1024 PC apply: TMA kernels (FPC_TIME_TMA_1024=1) vs the split kernels."""
import os, subprocess, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CASES = [("1d", 8191, 1024), ("2d", 127, 1024), ("1d", 4095, 1024)]
def child(tag):
    import numpy as np, torch
    import paper_2003_07020_b200 as fp
    out = {}
    for kind, n, nt in CASES:
        h, dt = 1.0 / (n + 1), 1.0 / nt
        jac = fp.RieszJacobian2D(1.3, 1.7, 1.0, 1.0, h, n) if kind == "2d" else fp.RieszJacobian1D(1.5, 1.0, h, n)
        op = fp.AllAtOnceOperator(fp.TimeStencil(nt), jac, dt)
        plan = fp.build_plan(fp.PreconditionerKind.generalized(), nt, dt, op)
        ns = n * n if kind == "2d" else n
        g = torch.Generator(device="cuda").manual_seed(7)
        b = torch.rand(nt * ns, dtype=torch.float64, device="cuda", generator=g) - 0.5
        y = torch.empty_like(b)
        fp.apply_inverse(plan, b, y)
        torch.cuda.synchronize()
        with fp.KernelProfile() as prof:
            for _ in range(5):
                fp.apply_inverse(plan, b, y)
        torch.cuda.synchronize()
        key = f"{kind}_{n}_{nt}"
        np.save(f"/tmp/t1k_{tag}_{key}.npy", y.cpu().numpy())
        out[key] = {k: round(1e3 * v[0] / v[1], 1) for k, v in prof.table.items()}
    print(json.dumps(out))
if len(sys.argv) > 1:
    child(sys.argv[1])
else:
    import numpy as np
    res = {}
    for tag, env in (("split", "0"), ("tma", "1")):
        r = subprocess.run([sys.executable, __file__, tag], env={**os.environ, "FPC_TIME_TMA_1024": env}, capture_output=True, text=True)
        if r.returncode != 0:
            print(r.stdout[-2000:], r.stderr[-2000:]); sys.exit(1)
        res[tag] = json.loads(r.stdout.strip().splitlines()[-1])
    for kind, n, nt in CASES:
        key = f"{kind}_{n}_{nt}"
        a, b = np.load(f"/tmp/t1k_split_{key}.npy"), np.load(f"/tmp/t1k_tma_{key}.npy")
        print(key, f"rel diff {np.linalg.norm(a-b)/np.linalg.norm(a):.2e}", "split", res["split"][key], "tma", res["tma"][key])
