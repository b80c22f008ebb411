import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2304_04980_b200 import GpuSchurOperator, GpuNestedJacobiPreconditioner, generators
K, N, T = [int(x) for x in sys.argv[1:4]]
ga = generators.config4(0, K=K, N=N, T=T)
r = np.random.default_rng(1).standard_normal(ga.offset.shape[0])
os.environ["GQ_CTA"] = "0"
op0 = GpuSchurOperator(ga, 2, 1); pc0 = GpuNestedJacobiPreconditioner(op0, 2, 1)
a0 = np.asarray(pc0.apply(r))
os.environ["GQ_CTA"] = "1"
op1 = GpuSchurOperator(ga, 2, 1); pc1 = GpuNestedJacobiPreconditioner(op1, 2, 1)
for env in [{}, {"GQ_CTA_PERSIST": "1"}, {"GQ_CTA_R_INNER": "2", "GQ_CTA_R_OUTER": "3"}, {"GQ_CTA_R_INNER": "4", "GQ_CTA_R_OUTER": "7"}]:
    for k in ("GQ_CTA_DBG", "GQ_CTA_R_INNER", "GQ_CTA_R_OUTER", "GQ_CTA_PERSIST"): os.environ.pop(k, None)
    os.environ.update(env)
    outs = [np.asarray(pc1.apply(r)) for _ in range(2)]
    for a1 in outs:
        d = np.abs(a1 - a0).reshape(T + 1, N, K, 2).max(axis=3)
        bad = np.argwhere(d > 1e-10 * np.abs(a0).max())
        res = {"rel": float(np.abs(a1 - a0).max() / np.abs(a0).max()), "nbad": int(len(bad))}
        if len(bad):
            t = bad[:, 0]; j = bad[:, 1]; i = bad[:, 2]
            c = (t - 1) // 40; w = ((t - 1) % 40) // 8
            res["warp_hist"] = np.bincount(w, minlength=5).tolist()
            res["c_hist"] = np.bincount(c, minlength=5).tolist()
            res["blk_hist"] = np.bincount(i // 2, minlength=16)[:20].tolist()
            vc = np.unique(np.stack([j // 2, c], 1), axis=0)
            res["n_items_bad"] = int(len(vc)); res["items"] = vc[:12].tolist()
        print(json.dumps(env), json.dumps(res), flush=True)
