"""Config 5 at full size: PCG to 1e-10 relative (S = L = 2), true residual, vs GQ_NO_CHAIN."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2304_04980_b200 import (GpuSchurOperator, GpuNestedJacobiPreconditioner, generators,
                                   pcg_solve, MaxIterationsExceeded)
ga = generators.config5(0)
rhs = torch.tensor(ga.offset, device="cuda", dtype=torch.float64)
tol = 1e-10 * float(rhs.abs().max())
for var in sys.argv[1:] or ["DEFAULT=1"]:
    for k in list(os.environ):
        if k.startswith("GQ_"): os.environ.pop(k)
    for kv in var.split(","):
        k, v = kv.split("="); os.environ["GQ_" + k] = v
    op = GpuSchurOperator(ga, 2, 2); pc = GpuNestedJacobiPreconditioner(op, 2, 2)
    v = torch.randn(op.dim, device="cuda", dtype=torch.float64)
    p1 = pc.apply(v)
    t0 = time.time()
    try:
        x, rep = pcg_solve(op, pc, rhs, tol=tol, max_steps=300)
    except MaxIterationsExceeded as e:
        x, rep = e.iterate, e.report
    torch.cuda.synchronize()
    res = float((op.apply(x) - rhs).abs().max() / rhs.abs().max())
    print(var, "steps", rep.steps, "conv", rep.converged, "time", round(time.time() - t0, 2), "true res", res,
          "precond|v|", float(p1.abs().max()), flush=True)
    if var == "DEFAULT=1": pref = p1.cpu()
    else: print("  precond rel diff vs default", float((p1.cpu() - pref).abs().max() / pref.abs().max()))
    del op, pc; torch.cuda.empty_cache()
