"""Per-instruction stall profile of one kernel from an ncu report (SASS page): the instructions
holding the most stall samples, and a running profile along the instruction stream in segments.
usage: python scripts/ncu_sass.py <rep> <kernel regex> [top] [segment]"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
seg = int(sys.argv[4]) if len(sys.argv) > 4 else 100
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if "Address" in r)
hdr = rows[hi]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
data = []
for r in rows[hi + 1:]:
    if len(r) < len(hdr):
        break  # next kernel instance
    try:
        w = float(r[ix["Warp Stall Sampling (All Samples)"]])
    except ValueError:
        continue
    data.append((w, r))
tot = sum(w for w, _ in data) or 1
print("instructions", len(data), "samples", tot)
agg = {s: sum(float(r[ix[s]] or 0) for _, r in data) for s in stalls}
print("stall mix:", ", ".join(f"{s[6:]} {100*v/tot:.0f}%" for s, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
print("-- top instructions")
for n, (w, r) in sorted(enumerate(data), key=lambda t: -t[1][0])[:top]:
    why = sorted(((float(r[ix[s]] or 0), s[6:]) for s in stalls), reverse=True)[:2]
    print(f"{100*w/tot:5.1f}% #{n:5d} {r[ix['Source']][:70]:70s} {why[0][1]}:{why[0][0]:.0f} {why[1][1]}:{why[1][0]:.0f}")
print(f"-- segments of {seg} instructions")
for s0 in range(0, len(data), seg):
    chunk = data[s0:s0 + seg]
    w = sum(c[0] for c in chunk)
    ops = {}
    for _, r in chunk:
        op = r[ix["Source"]].split()[0].split(".")[0] if r[ix["Source"]] else "?"
        if op.startswith("@"):
            op = r[ix["Source"]].split()[1].split(".")[0]
        ops[op] = ops.get(op, 0) + 1
    mix = " ".join(f"{k}{v}" for k, v in sorted(ops.items(), key=lambda kv: -kv[1])[:5])
    sm = {s: sum(float(r[ix[s]] or 0) for _, r in chunk) for s in stalls}
    why = sorted(sm.items(), key=lambda kv: -kv[1])[:2]
    print(f"{s0:5d} {100*w/tot:5.1f}%  {mix:40s} {why[0][0][6:]}:{100*why[0][1]/tot:.1f} {why[1][0][6:]}:{100*why[1][1]/tot:.1f}")
