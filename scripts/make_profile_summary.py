"""Write profiles/<tag>_summary.md (+ traffic.json) from an ncu --set full report and a launch list.

usage: python scripts/make_profile_summary.py <prof.ncu-rep> <launches.csv> <tag>
"""
import csv, io, json, os, subprocess, sys
from collections import defaultdict

rep, launches, tag = sys.argv[1], sys.argv[2], sys.argv[3]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
col = lambda r, name: r[hdr.index(name)] if name in hdr else ""
# map kernel names to the library's launch categories (bench.py roofline keys)
cats = [("k_matvec_split", "matvec_1d"), ("k_matvec_1d_split", "matvec_1d"), ("k_matvec_1d", "matvec_1d"), ("k_matvec_2d", "matvec_2d"),
        ("k_time_fwd", "time_fwd"), ("k_time_inv", "time_inv"), ("k_tau_solve_1d", "tau_solve_1d"),
        ("k_tau_2d", "tau_solve_2d"), ("k_update_dots", "update_dots"), ("k_dots2", "dots2"), ("k_update2", "update2"), ("k_dots", "dots"), ("k_update", "update")]
out = [f"# ncu summary `{tag}` (B200, `--set full --clock-control none`, config 1 bench)\n",
       "Per-kernel figures of one launch each (ncu replays: cold-cache, serialised).\n",
       "| kernel | time (us) | DRAM read (MB) | DRAM write (MB) | DRAM % peak | fp64 pipe % | L1/smem % | warps active % | regs | top stalls |",
       "|---|---|---|---|---|---|---|---|---|---|"]
traffic = {}
onchip = {}  # per category: the on-chip pipes that bound the FFT kernels (bench.py roofline.onchip)
for r in rows[2:]:
    name = col(r, "Kernel Name")
    st = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try:
                st.append((float(r[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(v for v, _ in st) or 1
    st.sort(reverse=True)
    rd, wr = float(col(r, "dram__bytes_read.sum") or 0), float(col(r, "dram__bytes_write.sum") or 0)
    unit_r = rows[1][hdr.index("dram__bytes_read.sum")]
    scale = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0}.get(unit_r, 1e6)
    out.append(f"| `{name.split('(')[0]}` | {col(r, 'gpu__time_duration.sum')} | {rd:.1f} | {wr:.1f} | "
               f"{float(col(r, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed') or 0):.1f} | "
               f"{float(col(r, 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active') or 0):.1f} | "
               f"{float(col(r, 'l1tex__throughput.avg.pct_of_peak_sustained_active') or 0):.1f} | "
               f"{float(col(r, 'sm__warps_active.avg.pct_of_peak_sustained_active') or 0):.1f} | "
               f"{col(r, 'launch__registers_per_thread')} | "
               + ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in st[:3]) + " |")
    for pat, cat in cats:
        if pat in name:
            traffic.setdefault(cat, (rd + wr) * scale)
            onchip.setdefault(cat, {
                "l1_smem_pct": float(col(r, 'l1tex__throughput.avg.pct_of_peak_sustained_active') or 0),
                "fp64_pipe_pct": float(col(r, 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active') or 0),
                "dram_pct": float(col(r, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed') or 0),
                "source": f"ncu --set full, profiles/{tag}_summary.md"})
            break
# launch list: share of device time per kernel family over the captured launches
share = defaultdict(float)
with open(launches) as f:
    lines = [l for l in f if not l.startswith("==")]
for r in csv.DictReader(io.StringIO("".join(lines))):
    if r.get("Metric Name") == "gpu__time_duration.sum":
        k = r["Kernel Name"].split("(")[0].replace("void ", "")
        v = float(r["Metric Value"].replace(",", ""))
        share[k] += v * (1e-3 if r.get("Metric Unit") in ("ns", "nsecond") else 1.0)
tot = sum(share.values()) or 1
out += ["", "## Launch list (ncu `gpu__time_duration.sum`, first 400 launches of `bench.py --steps 1 --warmup 1`)\n",
        "| kernel | total us | share |", "|---|---|---|"]
for k, v in sorted(share.items(), key=lambda kv: -kv[1]):
    out.append(f"| `{k}` | {v:.0f} | {100 * v / tot:.1f}% |")
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
open(os.path.join(ROOT, "profiles", f"{tag}_summary.md"), "w").write("\n".join(out) + "\n")
json.dump(traffic, open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)
json.dump(onchip, open(os.path.join(ROOT, "profiles", "onchip.json"), "w"), indent=1)
print("\n".join(out))
