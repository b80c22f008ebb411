"""Run a few PCGM steps at the headline size (target for ncu captures of the step kernels):
    ncu --set full -k regex:'k_stencil3|k_update|k_dirupdate|k_chain' --launch-skip 16 -c 8 python tools/stepprof.py
"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2304_04980_b200 import GpuSchurOperator, GpuNestedJacobiPreconditioner, _lib, generators
ga = generators.config4(0, N=int(os.environ.get("SP_N", "256")))
op = GpuSchurOperator(ga, 2, 2); pc = GpuNestedJacobiPreconditioner(op, 2, 2)
ctx = op._ctx; lib = ctx.lib
rhs = torch.tensor(ga.offset, device="cuda", dtype=torch.float64)
_lib.check(lib.gq_pcg_start(ctx.h, ctypes.c_void_p(rhs.data_ptr()), None, 1))
steps, conv = ctypes.c_int64(), ctypes.c_int32()
lib.gq_pcg_run(ctx.h, 1e-300, int(os.environ.get("STEPS", "4")), ctypes.byref(steps), ctypes.byref(conv))
torch.cuda.synchronize()
print("steps", steps.value)
