"""Two independent preconditioner applies (two contexts) back to back vs on two streams:
does the GPU have room for overlapping sweep kernels?"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2304_04980_b200 import GpuSchurOperator, GpuNestedJacobiPreconditioner, _lib, generators
ga = generators.config4(0)
ops = [GpuSchurOperator(ga, 2, 2) for _ in range(2)]
pcs = [GpuNestedJacobiPreconditioner(o, 2, 2) for o in ops]
sts = [torch.cuda.Stream() for _ in range(2)]
for o, s in zip(ops, sts):
    _lib.check(o._ctx.lib.gq_set_stream(o._ctx.h, ctypes.c_void_p(s.cuda_stream)))
v = torch.randn(ops[0].dim, device="cuda", dtype=torch.float64)
outs = [torch.empty_like(v) for _ in range(2)]
lib = ops[0]._ctx.lib
def apply(i):
    _lib.check(lib.gq_apply_precond(ops[i]._ctx.h, ctypes.c_void_p(v.data_ptr()), ctypes.c_void_p(outs[i].data_ptr())))
for _ in range(2): apply(0); apply(1)
torch.cuda.synchronize()
import time
for mode in ("seq", "seq", "seq"):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(10): apply(0); apply(1)
    torch.cuda.synchronize(); print(mode, (time.perf_counter() - t0) / 20 * 1e3, "ms per apply")
