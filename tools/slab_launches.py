"""A few native stage-slab steps at the headline (2 slabs in this process), for an ncu
launch list: python tools/slab_launches.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_04980_b200 import MaxIterationsExceeded  # noqa: E402
from paper_2304_04980_b200.generators import config4  # noqa: E402
from paper_2304_04980_b200.slab import SlabComm, SlabPcg  # noqa: E402

ga = config4()
rhs = torch.from_numpy(ga.offset).cuda()
s = SlabPcg(ga, comm=SlabComm(int(os.environ.get("SLABS", "2")), device=torch.device("cuda")),
            graph=False)
try:
    s.solve(rhs, tol=1e-300, max_steps=int(os.environ.get("STEPS", "3")))
except MaxIterationsExceeded as exc:
    print("steps", exc.report.steps, "res", exc.report.residual_inf_history[-1])
