"""n = 8 chain sweeps vs the CPU oracle on a mid-size config-5-like case, then config 5 timing."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2304_04980_b200 import GpuSchurOperator, GpuNestedJacobiPreconditioner, generators
from oracle.gridlq_oracle import Oracle
for (K, N, T) in [(8, 16, 20), (7, 10, 9)]:
    ga = generators.config5(0, K=K, N=N, T=T)
    op = GpuSchurOperator(ga, 2, 2); pc = GpuNestedJacobiPreconditioner(op, 2, 2)
    orc = Oracle(ga, 2, 2)
    v = np.random.default_rng(0).standard_normal(op.dim)
    a = np.asarray(pc.apply(v)); b = orc.apply_precond(v)
    print(K, N, T, "precond rel", np.max(np.abs(a - b)) / np.max(np.abs(b)), flush=True)
for (K, N, T) in [(8, 16, 20), (7, 10, 9), (5, 3, 4)]:
    ga = generators.config5(0, K=K, N=N, T=T)
    op = GpuSchurOperator(ga, 2, 2)
    orc = Oracle(ga, 2, 2)
    v = np.random.default_rng(1).standard_normal(op.dim)
    a = np.asarray(op.apply(v)); b = orc.apply_delta(v)
    print(K, N, T, "delta rel", np.max(np.abs(a - b)) / np.max(np.abs(b)), flush=True)
