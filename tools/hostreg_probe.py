"""Cost of cudaHostRegister / Unregister on a prefaulted 211 MB numpy array, and the D2H copy
into it (pinned in place) against the staged pageable path."""
import ctypes, time, numpy as np, torch
cudart = ctypes.CDLL("libcudart.so.12") if False else None
import torch.cuda
rt = torch.cuda.cudart()
n = 26345472
x = np.empty(n); x[::512] = 0.0
d = torch.randn(n, device="cuda", dtype=torch.float64)
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter()
    rc = rt.cudaHostRegister(x.ctypes.data, x.nbytes, 0)
    t1 = time.perf_counter()
    torch.from_numpy(x).copy_(d, non_blocking=False) if False else None
    h = torch.from_numpy(x)
    h.copy_(d); torch.cuda.synchronize()
    t2 = time.perf_counter()
    rt.cudaHostUnregister(x.ctypes.data)
    t3 = time.perf_counter()
    y = np.empty(n); y[::512] = 0.0
    t4 = time.perf_counter()
    torch.from_numpy(y).copy_(d); torch.cuda.synchronize()
    t5 = time.perf_counter()
    print(f"register {1e3*(t1-t0):.1f} ms  copy(pinned in place) {1e3*(t2-t1):.1f} ms  unregister {1e3*(t3-t2):.1f} ms | pageable torch copy {1e3*(t5-t4):.1f} ms", rc)
