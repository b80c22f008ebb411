"""Run every BASELINE.json configuration through the device PCGM and record steps, time and
steps/s (config 5: the S x L sweep with iterations to 1e-10 * ||omega~||_inf; L = 1 is refused
by the reference, nested_jacobi.py:112-116).  Writes one JSON document to stdout.

    python tools/configs_report.py > profiles/r01b/configs.json
"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2304_04980_b200 import (GpuNestedJacobiPreconditioner, GpuSchurOperator,
                                   MaxIterationsExceeded, generators, pcg_solve)


def run(ga, S, L, tol=None, rel_tol=None, max_steps=None):
    t0 = time.perf_counter()
    op = GpuSchurOperator(ga, L, S)
    pc = GpuNestedJacobiPreconditioner(op, L, S)
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    rhs = torch.tensor(ga.offset, device="cuda", dtype=torch.float64)
    if rel_tol is not None:
        tol = rel_tol * float(rhs.abs().max())
    try:                                   # warm-up (graph capture, first launches)
        pcg_solve(op, pc, rhs, tol=tol, max_steps=2)
    except MaxIterationsExceeded:
        pass
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    try:
        x, rep = pcg_solve(op, pc, rhs, tol=tol, max_steps=max_steps)
    except MaxIterationsExceeded as exc:
        x, rep = exc.iterate, exc.report
    torch.cuda.synchronize()
    solve = time.perf_counter() - t0
    res = float((op.apply(x) - rhs).abs().max() / rhs.abs().max())
    out = dict(dim=op.dim, S=S, L=L, tol=tol, steps=rep.steps, converged=bool(rep.converged),
               solve_s=round(solve, 4), steps_per_s=round(rep.steps / solve, 2),
               setup_s=round(setup, 3), final_res_inf=rep.residual_inf_history[-1],
               true_rel_residual=res)
    del op, pc
    torch.cuda.empty_cache()
    return out


rep = {"device": torch.cuda.get_device_name(0), "note": "device vectors in/out; solve_s is the "
       "wall clock of pcg_solve (initial preconditioner apply + steps + reads), setup excluded"}
rep["config1"] = run(generators.config1(0), 2, 2, tol=1e-300, max_steps=50)
rep["config2"] = run(generators.config2(0), 2, 2, rel_tol=1e-10)
rep["config3"] = [run(generators.config3(0), 3, L, tol=1e-300, max_steps=200) for L in (2, 4)]
rep["config4"] = run(generators.config4(0), 2, 2, tol=1e-300, max_steps=100)
ga5 = generators.config5(0)
rep["config5"] = {"L=1": "refused by the reference (odd inner budget, nested_jacobi.py:112-116)"}
for S in (1, 2, 4):
    for L in (2, 4):
        rep["config5"][f"S={S},L={L}"] = run(ga5, S, L, rel_tol=1e-10, max_steps=2000)
print(json.dumps(rep, indent=1))
