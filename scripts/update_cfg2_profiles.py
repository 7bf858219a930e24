"""Update profiles/traffic.json, profiles/onchip.json (config 2 entries bench.py reads) and append
a section to profiles/r2_summary.md from the raw CSV page of an `ncu --set full` capture of
scripts/op_once.py 2 (one matvec + one PC apply).
usage: python scripts/update_cfg2_profiles.py <raw.csv> <tag>"""
import csv, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rows = list(csv.reader(open(sys.argv[1])))
tag = sys.argv[2]
hdr, units = rows[0], rows[1]
W = "cfg2_2d_255sq_x512_g1.3_1.7"
def col(r, n): return r[hdr.index(n)]
def mb(r, n):
    u = units[hdr.index(n)]
    return float(col(r, n)) * {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0}[u]
cat = lambda name: ("matvec_2d" if "k_mv_" in name else "tau_solve_2d" if ("k_dst_rows" in name or "k_tau_cols" in name)
                    else "time_fwd" if "k_time_fwd" in name else "time_inv" if "k_time_inv" in name else None)
traffic, onchip, lines = {}, {}, []
for r in rows[2:]:
    name = col(r, "Kernel Name")
    c = cat(name)
    if not c:
        continue
    short = name.split("(")[0].replace("void ", "").replace("fpc::", "")
    by = mb(r, "dram__bytes_read.sum") + mb(r, "dram__bytes_write.sum")
    traffic[c] = traffic.get(c, 0.0) + by
    st = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try: st.append((float(r[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError: pass
    tot = sum(v for v, _ in st) or 1
    st.sort(reverse=True)
    k = {"us_ncu": round(float(col(r, "gpu__time_duration.sum")), 1),
         "fp64_pipe_pct": round(float(col(r, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")), 1),
         "l1tex_pct": round(float(col(r, "l1tex__throughput.avg.pct_of_peak_sustained_active")), 1),
         "dram_pct": round(float(col(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")), 1),
         "warps_active_pct": round(float(col(r, "sm__warps_active.avg.pct_of_peak_sustained_active")), 1)}
    onchip.setdefault(c, {"kernels": {}, "source": f"ncu --set full, profiles/r2_summary.md ({tag})"})["kernels"].setdefault(short, k)
    lines.append(f"| `{short}` | {k['us_ncu']} | {mb(r, 'dram__bytes_read.sum')/1e6:.1f} | {mb(r, 'dram__bytes_write.sum')/1e6:.1f} | "
                 f"{k['dram_pct']} | {k['fp64_pipe_pct']} | {k['l1tex_pct']} | {k['warps_active_pct']} | "
                 f"{col(r, 'launch__registers_per_thread')} | " + ", ".join(f"{n} {100*v/tot:.0f}%" for v, n in st[:4]) + " |")
for fn, upd in (("traffic.json", traffic), ("onchip.json", onchip)):
    p = os.path.join(ROOT, "profiles", fn)
    d = json.load(open(p))
    d.setdefault(W, {}).update(upd)
    d[W].pop("tau_solve_2d_note", None)
    json.dump(d, open(p, "w"), indent=1)
with open(os.path.join(ROOT, "profiles", "r2_summary.md"), "a") as f:
    f.write(f"\n## `{tag}`: config 2, one matvec + one PC apply (`scripts/op_once.py 2`), per launch\n\n"
            "| kernel | time (us) | DRAM read (MB) | DRAM write (MB) | DRAM % | fp64 pipe % | L1/shared % | warps active % | regs | top stalls |\n"
            "|---|---|---|---|---|---|---|---|---|---|\n" + "\n".join(lines) + "\n")
print(json.dumps(traffic), "\n".join(lines))
