"""Stall breakdown + top SASS lines per kernel of an .ncu-rep: python tools/ncu_stalls.py rep [ntop]"""
import csv, io, subprocess, sys
from collections import Counter
rep = sys.argv[1]; ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 20
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
for r in rows[2:]:
    items = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try: items.append((float(r[i]), h[len("smsp__pcsamp_warps_issue_stalled_"):]))
            except ValueError: pass
    tot = sum(v for v, _ in items) or 1
    print(r[hdr.index("ID")], r[hdr.index("Kernel Name")][:40], sorted([(round(v / tot * 100, 1), h) for v, h in items], reverse=True)[:8])
    for k in ["smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__cycles_elapsed.avg"]:
        if k in hdr: print("   ", k, r[hdr.index(k)])
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
blocks, cur = [], None
for l in src.split("\n"):
    if l.startswith('"Kernel Name"'):
        cur = [l]; blocks.append(cur)
    elif cur is not None: cur.append(l)
seen = set()
for b in blocks:
    if b[0] in seen: continue
    seen.add(b[0])
    rs = list(csv.DictReader(b[1:]))
    tot = sum(int(x["Instructions Executed"] or 0) for x in rs)
    print(b[0][15:90], "warp-instr", tot)
    c = Counter()
    for x in rs:
        s = x["Source"].strip().split()
        if not s: continue
        op = s[1] if s[0].startswith("@") else s[0]
        c[op.split(".")[0]] += int(x["Instructions Executed"] or 0)
    print("   ", [(k, round(v / tot * 100, 1)) for k, v in c.most_common(16)])
    for x in sorted(rs, key=lambda x: -int(x["Warp Stall Sampling (All Samples)"] or 0))[:ntop]:
        print(f'    {x["Address"][-5:]} {int(x["Warp Stall Sampling (All Samples)"]):6d} {int(x["Instructions Executed"]):9d} {x["Source"].strip()[:90]}')
