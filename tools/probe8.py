import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["GQ_EXP"] = "7"
import numpy as np, torch
from paper_2304_04980_b200 import GpuSchurOperator, GpuNestedJacobiPreconditioner, generators, _lib
ga = generators.config4(0)
op = GpuSchurOperator(ga); pc = GpuNestedJacobiPreconditioner(op, 2, 2)
v = torch.randn(op.dim, device="cuda", dtype=torch.float64)
lib = _lib.load()
# pair solve only (one non-inner sweep) to isolate
for _ in range(2): q = pc.apply(v)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * 800)()
lib.gq_debug_read(buf, 800)
a = np.array(buf[:800]).reshape(200, 4)
print("fill empty-wait, consumer full-wait, consumer timestamp")
print(a[:24, :3])
ts = a[:128, 2]
print("consumer block period (median cycles):", np.median(np.diff(ts[1:127])))
print("median empty-wait", np.median(a[8:128, 0]), "median full-wait", np.median(a[8:128, 1]))
