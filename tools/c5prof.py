"""A few PCGM steps of config 5 (n = 8) for ncu captures of the n = 8 kernels."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2304_04980_b200 import GpuSchurOperator, GpuNestedJacobiPreconditioner, _lib, generators
ga = generators.config5(0)
op = GpuSchurOperator(ga, 2, 2); pc = GpuNestedJacobiPreconditioner(op, 2, 2)
ctx = op._ctx; lib = ctx.lib
rhs = torch.tensor(ga.offset, device="cuda", dtype=torch.float64)
_lib.check(lib.gq_pcg_start(ctx.h, ctypes.c_void_p(rhs.data_ptr()), None, 1))
steps, conv = ctypes.c_int64(), ctypes.c_int32()
lib.gq_pcg_run(ctx.h, 1e-300, int(os.environ.get("STEPS", "2")), ctypes.byref(steps), ctypes.byref(conv))
torch.cuda.synchronize()
print("steps", steps.value)
