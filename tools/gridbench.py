"""Time the Delta apply (grid stencil) alone at the headline size: ms per launch."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2304_04980_b200 import GpuSchurOperator, generators
ga = generators.config4(0)
op = GpuSchurOperator(ga, 2, 2)
v = torch.randn(op.dim, device="cuda", dtype=torch.float64)
for _ in range(2): op.apply(v)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(10): op.apply(v)
e1.record(); torch.cuda.synchronize()
print(json.dumps({"ex": os.environ.get("GQ_GRID_EX", "0"), "ms_per_apply_incl_transposes": round(e0.elapsed_time(e1) / 10, 4)}))
