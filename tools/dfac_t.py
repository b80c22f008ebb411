import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2304_04980_b200 import GpuSchurOperator, generators
from oracle.gridlq_oracle import Oracle
sz = [int(a) for a in sys.argv[1:4]]
ga = generators.config4(0, K=sz[0], N=sz[1], T=sz[2])
t0 = time.time()
op = GpuSchurOperator(ga, 2, 2)
print("setup", time.time() - t0, flush=True)
v = np.random.default_rng(0).standard_normal(op.dim)
y = op.apply(v)
torch.cuda.synchronize()
print("apply ok", time.time() - t0, flush=True)
if op.dim < 2_000_000:
    ref = Oracle(ga, 2, 2).apply_delta(v)
    print("rel", np.max(np.abs(y - ref)) / np.max(np.abs(ref)), flush=True)
