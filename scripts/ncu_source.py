"""Top stall instructions of one kernel in an ncu report (SASS + CUDA source line)."""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass,cuda"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
# find header row
hi = next(i for i, r in enumerate(rows) if "Address" in r or "# Address" in r)
hdr = rows[hi]
ia = hdr.index("Address") if "Address" in hdr else hdr.index("# Address")
isrc = hdr.index("Source")
iw = hdr.index("Warp Stall Sampling (All Samples)")
data, seen, tot = [], set(), 0.0
for r in rows[hi + 1:]:
    if len(r) <= iw:
        continue
    try:
        w = float(r[iw])
    except ValueError:
        continue
    key = (r[ia], r[isrc])
    if key in seen:
        continue
    seen.add(key)
    tot += w
    data.append((w, r[ia], r[isrc]))
data.sort(reverse=True)
print("total samples", tot)
for w, a, s in data[:top]:
    print(f"{100*w/tot:5.1f}% {a:>18} {s[:120]}")
