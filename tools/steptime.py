"""Device time per PCGM step (captured graph) at the headline size for env variants, each in
its own context, interleaved over several rounds: python tools/steptime.py "" NO_FUSE_R=1 ..."""
import ctypes, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2304_04980_b200 import GpuSchurOperator, GpuNestedJacobiPreconditioner, _lib, generators

ga = generators.config4(0)
rhs = torch.tensor(ga.offset, device="cuda", dtype=torch.float64)
variants = sys.argv[1:] or [""]
res = {v: [] for v in variants}
ops = {}


def set_env(var):
    # the library reads GQ_* both at setup and when it captures the step graph (first run)
    env = dict(kv.split("=") for kv in var.split(",") if kv)
    for k in list(os.environ):
        if k.startswith("GQ_"): os.environ.pop(k)
    for k, val in env.items(): os.environ["GQ_" + k] = val


for var in variants:
    set_env(var)
    op = GpuSchurOperator(ga, 2, 2)
    pc = GpuNestedJacobiPreconditioner(op, 2, 2)
    st = torch.cuda.Stream()
    _lib.check(op._ctx.lib.gq_set_stream(op._ctx.h, ctypes.c_void_p(st.cuda_stream)))
    ops[var] = (op, pc, st)
steps, conv = ctypes.c_int64(), ctypes.c_int32()
for rnd in range(int(os.environ.get("ROUNDS", "3"))):
    for var in variants:
        set_env(var)
        op, pc, st = ops[var]
        ctx = op._ctx; lib = ctx.lib
        _lib.check(lib.gq_pcg_start(ctx.h, ctypes.c_void_p(rhs.data_ptr()), None, 1))
        lib.gq_pcg_run(ctx.h, 1e-300, 3, ctypes.byref(steps), ctypes.byref(conv))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(st)
        lib.gq_pcg_run(ctx.h, 1e-300, 53, ctypes.byref(steps), ctypes.byref(conv))
        e1.record(st); torch.cuda.synchronize()
        res[var].append(e0.elapsed_time(e1) / 50)
for var in variants:
    print(json.dumps({"env": var, "ms_per_step": [round(x, 4) for x in res[var]],
                      "steps_per_s": round(1000 / min(res[var]), 1)}), flush=True)
