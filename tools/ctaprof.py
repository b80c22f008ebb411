"""One L=2,S=1 preconditioner apply at the headline size (ncu target for the chain sweeps)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2304_04980_b200 import GpuSchurOperator, GpuNestedJacobiPreconditioner, generators
ga = generators.config4(0)
op = GpuSchurOperator(ga, 2, 1); pc = GpuNestedJacobiPreconditioner(op, 2, 1)
v = torch.randn(op.dim, device="cuda", dtype=torch.float64)
for _ in range(int(os.environ.get("REPS", "2"))): pc.apply(v)
torch.cuda.synchronize()
print("ok")
