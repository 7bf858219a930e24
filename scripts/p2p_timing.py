"""Peer-store exchange kernel (kernels_p2p.cu) at config-1 shapes, all G destination buffers on this
one GPU (simulated ranks, run one after the other): the kernel's own access-pattern efficiency
against the HBM copy roofline (bytes = one read + one write per element).  NVLink is not exercised.
usage: python scripts/p2p_timing.py [G]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2003_07020_b200 as fp
from paper_2003_07020_b200.distributed import CudaShardKernels, offsets, split_counts

G = int(sys.argv[1]) if len(sys.argv) > 1 else 8
nt, ns = 2048, 8191
H, nt_loc = nt // 2 + 1, nt // G
cs, hs = split_counts(ns, G), split_counts(H, G)
co, ho = offsets(cs), offsets(hs)
ctx = fp.Context(0, torch.cuda.current_stream())
op = fp.AllAtOnceOperator(fp.TimeStencil(16), fp.RieszJacobian1D(1.5, 1.0, 1 / 16, 15), 1 / 16, ctx)
k = CudaShardKernels(op, None)
dev = torch.device("cuda", 0)
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json"))).get("hbm_gbs", 6541.5) \
    if os.path.exists(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) else 6541.5
cases = {
    # name: (src doubles, dst doubles per rank, es, split_cols, off, stride, row_base, col_base, rows, cols)
    "time_to_space": (nt_loc * ns, [nt * c for c in cs], 1, True, co, cs, lambda r: r * nt_loc, lambda r: 0,
                      lambda r: (nt_loc, ns)),
    "space_to_freq": (2 * H * max(cs), [2 * h * ns for h in hs], 2, False, ho, [ns] * G, lambda r: 0,
                      lambda r: co[r], lambda r: (H, cs[r])),
}
out = {}
for name, (nsrc, ndst, es, split_cols, off, stride, rb, cb, rc) in cases.items():
    src = torch.randn(nsrc, dtype=torch.float64, device=dev)
    dst = [torch.empty(n, dtype=torch.float64, device=dev) for n in ndst]
    ptrs = [d.data_ptr() for d in dst]
    flush = torch.empty(64 << 20, dtype=torch.float64, device=dev)  # 512 MB > L2 between launches

    def step(r):
        rows, cols = rc(r)
        k.scatter_p2p(src, rows, cols, es, split_cols, ptrs, off, stride, rb(r), cb(r))

    for r in range(G):
        step(r)
    torch.cuda.synchronize()
    t = 0.0
    byt = 0
    for r in range(G):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        step(r)
        e1.record()
        torch.cuda.synchronize()
        t += e0.elapsed_time(e1) * 1e-3
        rows, cols = rc(r)
        byt += 2 * 8 * es * rows * cols
    out[name] = {"G": G, "us_per_rank": 1e6 * t / G, "GBs": byt / t / 1e9, "frac_hbm": byt / t / 1e9 / peak,
                 "bytes_per_rank": byt / G}
print(json.dumps({"kernel": "k_p2p_scatter", "config": "cfg1 8191x2048", "destinations": "local (simulated ranks)",
                  "peak_hbm_gbs": peak, "cases": out}))
