"""Steps/s of the stage-slab PCGM (paper_2304_04980_b200/slab.py) at the headline config,
with all slabs in this process on one GPU, against the one-context graph solve.
Usage: python tools/slabtime.py [slabs ...]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_04980_b200 import (GpuNestedJacobiPreconditioner, GpuSchurOperator,  # noqa: E402
                                   MaxIterationsExceeded, pcg_solve)
from paper_2304_04980_b200.generators import config4  # noqa: E402
from paper_2304_04980_b200.slab import SlabComm, SlabPcg  # noqa: E402

STEPS = int(os.environ.get("STEPS", "40"))
ga = config4()
rhs = torch.from_numpy(ga.offset).cuda()


def timed(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    try:
        fn()
    except MaxIterationsExceeded:
        pass
    torch.cuda.synchronize()
    return time.perf_counter() - t0


op = GpuSchurOperator(ga)
pc = GpuNestedJacobiPreconditioner(op)
timed(lambda: pcg_solve(op, pc, rhs, tol=1e-300, max_steps=3))
t = timed(lambda: pcg_solve(op, pc, rhs, tol=1e-300, max_steps=STEPS))
print({"mode": "graph", "steps": STEPS, "ms_per_step": round(1e3 * t / STEPS, 3)}, flush=True)
del op, pc
for p in [int(a) for a in sys.argv[1:]] or [1, 2, 4]:
    for native, graph in ((True, True), (True, False), (False, None)):
        s = SlabPcg(ga, comm=SlabComm(p, device=torch.device("cuda")), native=native, graph=graph)
        timed(lambda: s.solve(rhs, tol=1e-300, max_steps=3))
        per = []
        for _ in range(3):
            if native:       # CUDA events around the steps after the first 3 (slab.py)
                s.time_from = 3
                timed(lambda: s.solve(rhs, tol=1e-300, max_steps=3 + STEPS))
                per.append(s.last_timed[1] / STEPS)
            else:            # composed driver: difference of two solves
                t3 = timed(lambda: s.solve(rhs, tol=1e-300, max_steps=3))
                t = timed(lambda: s.solve(rhs, tol=1e-300, max_steps=3 + STEPS))
                per.append(1e3 * (t - t3) / STEPS)
        print({"mode": "slabs", "slabs": p, "native": native, "graph": graph, "steps": STEPS,
               "ms_per_step": round(sorted(per)[1], 3)}, flush=True)
        del s
    torch.cuda.empty_cache()
