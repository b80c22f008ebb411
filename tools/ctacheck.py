"""CTA/TMA chain sweeps vs the per-warp chain sweeps: preconditioner applies on several
problems (max rel diff) and headline timings.  python tools/ctacheck.py"""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2304_04980_b200 import GpuSchurOperator, GpuNestedJacobiPreconditioner, generators


def make(ga, L, S, cta):
    os.environ["GQ_CTA"] = "1" if cta else "0"
    op = GpuSchurOperator(ga, L, S)
    return op, GpuNestedJacobiPreconditioner(op, L, S)


def timed(pc, v, n=10):
    for _ in range(2): pc.apply(v)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n): pc.apply(v)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


out = {}
cases = [("c1", generators.config1(0)), ("c2", generators.config2(0)),
         ("oddk", generators.msd_case(7, 6, 13, 0)), ("t3", generators.msd_case(6, 4, 3, 0)),
         ("c4r", generators.config4(0, K=32, N=32, T=90))]
for name, ga in cases:
    for (L, S) in [(2, 1), (2, 2), (4, 2)]:
        r = np.random.default_rng(1).standard_normal(ga.offset.shape[0])
        op0, pc0 = make(ga, L, S, False)
        op1, pc1 = make(ga, L, S, True)
        a0 = np.asarray(pc0.apply(r)); a1 = np.asarray(pc1.apply(r))
        out[f"{name}_L{L}S{S}"] = float(np.max(np.abs(a1 - a0)) / np.max(np.abs(a0)))
print(json.dumps(out), flush=True)
ga = generators.config4(0)
res = {}
for cta in (False, True):
    for (L, S) in [(2, 1), (4, 1), (2, 2)]:
        op, pc = make(ga, L, S, cta)
        v = torch.randn(op.dim, device="cuda", dtype=torch.float64)
        res[f"{'cta' if cta else 'warp'}_L{L}S{S}"] = round(timed(pc, v), 4)
        if cta and (L, S) == (2, 2):
            op0, pc0 = make(ga, L, S, False)
            a0 = pc0.apply(v); a1 = pc.apply(v)
            res["headline_rel"] = float((a1 - a0).abs().max() / a0.abs().max())
        del op, pc
        torch.cuda.empty_cache()
print(json.dumps(res), flush=True)
