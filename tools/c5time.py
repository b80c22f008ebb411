"""Config 5 (n = 8) PCGM step time under env variants (each variant in its own context)."""
import ctypes, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2304_04980_b200 import GpuSchurOperator, GpuNestedJacobiPreconditioner, _lib, generators
ga = generators.config5(0)
rhs = torch.tensor(ga.offset, device="cuda", dtype=torch.float64)
for var in sys.argv[1:] or [""]:
    env = dict(kv.split("=") for kv in var.split(",") if kv)
    for k in list(os.environ):
        if k.startswith("GQ_"): os.environ.pop(k)
    for k, v in env.items(): os.environ["GQ_" + k] = v
    op = GpuSchurOperator(ga, 2, 2); pc = GpuNestedJacobiPreconditioner(op, 2, 2)
    ctx = op._ctx; lib = ctx.lib
    st = torch.cuda.Stream(); _lib.check(lib.gq_set_stream(ctx.h, ctypes.c_void_p(st.cuda_stream)))
    _lib.check(lib.gq_pcg_start(ctx.h, ctypes.c_void_p(rhs.data_ptr()), None, 1))
    steps, conv = ctypes.c_int64(), ctypes.c_int32()
    lib.gq_pcg_run(ctx.h, 1e-300, 2, ctypes.byref(steps), ctypes.byref(conv))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(st); lib.gq_pcg_run(ctx.h, 1e-300, 7, ctypes.byref(steps), ctypes.byref(conv)); e1.record(st)
    torch.cuda.synchronize()
    nk = lib.gq_launches_per_step(ctx.h); buf = (ctypes.c_float * nk)()
    lib.gq_profile_steps(ctx.h, 2, buf, nk)
    names = [lib.gq_kernel_name(ctx.h, i).decode() for i in range(nk)]
    print(json.dumps({"env": var, "ms_per_step": round(e0.elapsed_time(e1) / 5, 3),
                      "kernels": {n: round(buf[i] / 2, 3) for i, n in enumerate(names)}}), flush=True)
    del op, pc; torch.cuda.empty_cache()
