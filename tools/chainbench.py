"""Time preconditioner applies at the headline size for chain-kernel experiments:
L=2,S=1 (outer + inner sweep) and L=... ; prints ms per apply (includes layout transposes)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2304_04980_b200 import GpuSchurOperator, GpuNestedJacobiPreconditioner, generators
ga = generators.config4(0)
op = GpuSchurOperator(ga, 2, 1)
v = torch.randn(op.dim, device="cuda", dtype=torch.float64)
res = {}
for L in (2, 4):
    pc = GpuNestedJacobiPreconditioner(op, L, 1)
    for _ in range(2): pc.apply(v)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5): pc.apply(v)
    e1.record(); torch.cuda.synchronize()
    res[f"L{L}"] = round(e0.elapsed_time(e1) / 5, 4)
# L4 - L2 = 2 inner sweeps
res["inner_sweep_est"] = round((res["L4"] - res["L2"]) / 2, 4)
res["outer_sweep_est"] = round(res["L2"] - res["inner_sweep_est"], 4)   # + transposes
print(json.dumps({"exp": os.environ.get("GQ_CHAIN_EX", os.environ.get("GQ_CHAIN_EXP", "0")), **res}))
