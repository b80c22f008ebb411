"""Time one preconditioner apply (S=L=2: 4 sweeps + outer rhs) at the headline size."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2304_04980_b200 import GpuSchurOperator, GpuNestedJacobiPreconditioner, generators
ga = generators.config4(0)
op = GpuSchurOperator(ga); pc = GpuNestedJacobiPreconditioner(op, 2, 2)
v = torch.randn(op.dim, device="cuda", dtype=torch.float64)
for _ in range(2): pc.apply(v)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
n = 10
e0.record()
for _ in range(n): pc.apply(v)
e1.record(); torch.cuda.synchronize()
env = {k: v for k, v in os.environ.items() if k.startswith("GQ_")}
print(json.dumps({"env": env, "ms_per_apply": e0.elapsed_time(e1) / n}))
