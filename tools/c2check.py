"""GQ_CHAIN2C=1 (CTA-shared factor sweeps, n = 2) against the default sweeps: preconditioner
applies on several shapes (max rel diff)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2304_04980_b200 import GpuSchurOperator, GpuNestedJacobiPreconditioner, generators
for (K, N, T) in [(4, 4, 20), (7, 6, 13), (32, 32, 90), (256, 256, 200)]:
    ga = generators.config4(0, K=K, N=N, T=T)
    v = torch.tensor(np.random.default_rng(1).standard_normal(ga.offset.shape[0]), device="cuda")
    res = []
    for flag in ("0", "1"):
        os.environ["GQ_CHAIN2C"] = flag
        op = GpuSchurOperator(ga, 2, 2); pc = GpuNestedJacobiPreconditioner(op, 2, 2)
        res.append(pc.apply(v).cpu().numpy())
        del op, pc; torch.cuda.empty_cache()
    print(K, N, T, "rel", np.max(np.abs(res[1] - res[0])) / np.max(np.abs(res[0])), flush=True)
