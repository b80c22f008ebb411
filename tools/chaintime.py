"""Headline timings of the per-warp chain sweeps under env variants (each variant in its own
context): ms per preconditioner apply at L=2,S=1 and L=4,S=1 -> inner / outer estimates."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2304_04980_b200 import GpuSchurOperator, GpuNestedJacobiPreconditioner, generators


def timed(pc, v, n=10):
    for _ in range(2): pc.apply(v)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n): pc.apply(v)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


ga = generators.config4(0, T=int(os.environ.get("CT_T", "200")))
v = None
for var in (sys.argv[1:] or [""]):
    env = dict(kv.split("=") for kv in var.split(",") if kv)
    for k in list(os.environ):
        if k.startswith("GQ_"): os.environ.pop(k)
    for k, val in env.items(): os.environ["GQ_" + k] = val
    op = GpuSchurOperator(ga, 2, 1)
    if v is None: v = torch.randn(op.dim, device="cuda", dtype=torch.float64)
    pcs = {L: GpuNestedJacobiPreconditioner(op, L, 1) for L in (2, 4)}
    t2 = timed(pcs[2], v); t4 = timed(pcs[4], v)
    inner = (t4 - t2) / 2
    print(json.dumps({"env": env, "L2": round(t2, 4), "L4": round(t4, 4), "inner": round(inner, 4),
                      "outer+tr": round(t2 - inner, 4)}), flush=True)
    del op, pcs
    torch.cuda.empty_cache()
