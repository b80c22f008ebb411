"""Per-instruction stall attribution of an ncu report (source page, SASS), read here:
    python tools/ncu_src.py gpurun_out/x.ncu-rep [reason] [top]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
reason = sys.argv[2] if len(sys.argv) > 2 else None
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {c: 0 for c in cols}
recs = []
for k, r in enumerate(rows[2:]):
    try:
        v = {c: int(r[hdr.index(c)] or 0) for c in cols}
    except ValueError:
        continue
    for c in cols:
        tot[c] += v[c]
    recs.append((k, r[hdr.index("Source")].strip(), v, int(r[hdr.index("Instructions Executed")] or 0)))
S = sum(tot.values())
print("totals:", ", ".join(f"{c[6:]} {100*v/S:.1f}%" for c, v in sorted(tot.items(), key=lambda kv: -kv[1]) if v))
key = ("stall_" + reason) if reason else None
recs.sort(key=lambda x: -(x[2][key] if key else sum(x[2].values())))
for k, src, v, ex in recs[:top]:
    s = v[key] if key else sum(v.values())
    print(f"{k:5d} {s:6d} {ex:9d}  {src[:80]}")
