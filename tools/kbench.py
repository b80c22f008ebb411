"""Time one preconditioner apply (4 sweeps + outer rhs) at the headline size."""
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
e0.record(); n = 5
for _ in range(n): pc.apply(v)
e1.record(); torch.cuda.synchronize()
print(json.dumps({"exp": os.environ.get("GQ_EXP", "0"), "v": os.environ.get("GQ_SWEEP_V", "8"), "ms_per_apply": e0.elapsed_time(e1) / n}))
