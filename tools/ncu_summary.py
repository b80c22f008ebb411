"""Summarise an .ncu-rep (details page) into per-kernel key metrics: python tools/ncu_summary.py rep [pattern...]"""
import csv, io, subprocess, sys, json
rep = sys.argv[1]
pats = sys.argv[2:] or ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "L1/TEX Hit Rate",
                        "Registers Per Thread", "Achieved Occupancy", "Executed Ipc Active", "Issue Slots Busy",
                        "Warp Cycles Per Issued Instruction", "No Eligible", "Theoretical Occupancy",
                        "Dynamic Shared Memory Per Block", "Grid Size", "Compute (SM) Throughput"]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.DictReader(io.StringIO(out)))
res = {}
for r in rows:
    key = f'{r["ID"]}:{r["Kernel Name"].split("(")[0]}'
    for p in pats:
        if r["Metric Name"] == p or (p.endswith("*") and r["Metric Name"].startswith(p[:-1])):
            res.setdefault(key, {})[r["Metric Name"]] = f'{r["Metric Value"]} {r["Metric Unit"]}'
print(json.dumps(res, indent=1))
