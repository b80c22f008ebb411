import time, torch, numpy as np, sys
sys.path.insert(0, '/root/repo')
from paper_2304_04980_b200 import MaxIterationsExceeded
from paper_2304_04980_b200.generators import config4
from paper_2304_04980_b200.slab import SlabComm, SlabPcg
ga = config4()
s = SlabPcg(ga, comm=SlabComm(1, device=torch.device('cuda')))
rhs_host = torch.from_numpy(ga.offset.copy()).pin_memory().numpy()
def T(f):
    torch.cuda.synchronize(); t=time.perf_counter(); r=f(); torch.cuda.synchronize(); return r, 1e3*(time.perf_counter()-t)
for rep in range(2):
    _, t_up = T(lambda: torch.as_tensor(rhs_host).to('cuda'))
    cpu = torch.as_tensor(rhs_host)
    _, t_fin = T(lambda: bool(torch.isfinite(cpu).all()))
    dev = torch.as_tensor(rhs_host).to('cuda')
    _, t_down = T(lambda: dev.cpu().numpy())
    def solve(n):
        try: s.solve(rhs_host, tol=1e-300, max_steps=n)
        except MaxIterationsExceeded: pass
    _, t1 = T(lambda: solve(1))
    _, t50 = T(lambda: solve(50))
    print(f"up {t_up:.1f} ms  isfinite(cpu) {t_fin:.1f}  down {t_down:.1f}  solve1 {t1:.1f}  solve50 {t50:.1f}")
