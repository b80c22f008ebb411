"""Where does the end-to-end pcg_solve time go at the headline size?"""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2304_04980_b200 import GpuSchurOperator, GpuNestedJacobiPreconditioner, _lib, generators, pcg_solve, MaxIterationsExceeded
ga = generators.config4(0)
op = GpuSchurOperator(ga, 2, 2); pc = GpuNestedJacobiPreconditioner(op, 2, 2)
ctx = op._ctx; lib = ctx.lib
rhs = torch.from_numpy(ga.offset.copy()).pin_memory().numpy()
K = 100
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _lib.check(lib.gq_pcg_start(ctx.h, rhs.ctypes.data, None, 1))
    t1 = time.perf_counter()
    steps, conv = ctypes.c_int64(), ctypes.c_int32()
    lib.gq_pcg_run(ctx.h, 1e-300, K, ctypes.byref(steps), ctypes.byref(conv))
    t2 = time.perf_counter()
    x = np.empty(op.dim)
    _lib.check(lib.gq_pcg_read(ctx.h, _lib.GQ_VEC_X, x.ctypes.data))
    t3 = time.perf_counter()
    xp = torch.empty(op.dim, dtype=torch.float64).pin_memory().numpy()
    t4 = time.perf_counter()
    _lib.check(lib.gq_pcg_read(ctx.h, _lib.GQ_VEC_X, xp.ctypes.data))
    t5 = time.perf_counter()
    t6 = time.perf_counter()
    try:
        pcg_solve(op, pc, rhs, tol=1e-300, max_steps=K)
    except MaxIterationsExceeded:
        pass
    t7 = time.perf_counter()
    print(f"start {1e3*(t1-t0):.1f} ms  run {1e3*(t2-t1):.1f} ms  read(pageable) {1e3*(t3-t2):.1f} ms  pin-alloc {1e3*(t4-t3):.1f} ms  read(pinned) {1e3*(t5-t4):.1f} ms  pcg_solve total {1e3*(t7-t6):.1f} ms")
