"""A/B at the headline: the one-context graph step (gq_pcg_run, as bench.py times it) against
the native stage-slab step with 1 slab (difference of two solves), same process."""
import ctypes
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_04980_b200 import (GpuNestedJacobiPreconditioner, GpuSchurOperator,  # noqa: E402
                                   MaxIterationsExceeded, _lib)
from paper_2304_04980_b200.generators import config4  # noqa: E402
from paper_2304_04980_b200.slab import SlabComm, SlabPcg  # noqa: E402

K = int(os.environ.get("STEPS", "50"))
ga = config4()
rhs = torch.from_numpy(ga.offset).cuda()
op = GpuSchurOperator(ga)
pc = GpuNestedJacobiPreconditioner(op)
lib, h = op._ctx.lib, op._ctx.h
st = torch.cuda.Stream()
_lib.check(lib.gq_set_stream(h, ctypes.c_void_p(st.cuda_stream)))
steps, conv = ctypes.c_int64(), ctypes.c_int32()
for rep in range(3):
    _lib.check(lib.gq_pcg_start(h, ctypes.c_void_p(rhs.data_ptr()), None, 1))
    lib.gq_pcg_run(h, 1e-300, 3, ctypes.byref(steps), ctypes.byref(conv))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    lib.gq_pcg_run(h, 1e-300, 3 + K, ctypes.byref(steps), ctypes.byref(conv))
    e1.record(st)
    torch.cuda.synchronize()
    hist = (ctypes.c_double * (3 + K))()
    lib.gq_pcg_history(h, hist, 3 + K)
    print({"mode": "graph", "ms_per_step": round(e0.elapsed_time(e1) / K, 4),
           "steps": steps.value, "res_last": hist[2 + K]}, flush=True)
del op, pc
s = SlabPcg(ga, comm=SlabComm(1, device=torch.device("cuda")))


def run(n):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    try:
        s.solve(rhs, tol=1e-300, max_steps=n)
    except MaxIterationsExceeded as exc:
        rep = exc.report
    torch.cuda.synchronize()
    return time.perf_counter() - t0, rep


run(3)
for rep in range(3):
    ta, _ = run(3)
    tb, rb = run(3 + K)
    print({"mode": "slab1", "ms_per_step": round(1e3 * (tb - ta) / K, 4), "steps": rb.steps,
           "res_last": rb.residual_inf_history[-1]}, flush=True)
