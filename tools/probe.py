import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["GQ_EXP"] = "7"; os.environ["GQ_SWEEP_V"] = "6"
import numpy as np, torch
from paper_2304_04980_b200 import GpuSchurOperator, GpuNestedJacobiPreconditioner, generators, _lib
ga = generators.config4(0)
op = GpuSchurOperator(ga); pc = GpuNestedJacobiPreconditioner(op, 2, 2)
v = torch.randn(op.dim, device="cuda", dtype=torch.float64)
for _ in range(3): q = pc.apply(v)
torch.cuda.synchronize()
lib = _lib.load()
buf = (ctypes.c_longlong * 800)()
lib.gq_debug_read(buf, 800)
a = np.array(buf[:800]).reshape(200, 4)
print("issue, gmma+, wait, rest (cycles) per block, first 20 blocks:")
print(a[:20])
print("median over blocks 10..120:", np.median(a[10:120], axis=0))
