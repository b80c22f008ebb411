# which small shapes break the forced t-loop kernels (one subprocess per shape: CUDA errors are sticky)
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "one":
    sys.path.insert(0, ROOT)
    import numpy as np
    from paper_2304_04980_b200 import GpuSchurOperator, generators
    K, N, T = map(int, sys.argv[2:5])
    ga = generators.random_case(K, N, T, 2, 1, seed=0)
    v = np.random.default_rng(0).standard_normal(ga.offset.shape)
    op = GpuSchurOperator(ga, 2, 2)
    a = op.apply(v)
    b = op.apply_outer_coupling(v)
    np.save(f"/tmp/shape_{os.environ.get('GQ_DSTEP','0')}_{K}_{N}_{T}.npy", np.concatenate([a, b]))
    sys.exit(0)
for K in (3, 5, 33):
    for N in (3, 9):
        for T in (3, 4, 6, 19, 20):
            r = []
            for ds in ("1", "0"):
                p = subprocess.run([sys.executable, __file__, "one", str(K), str(N), str(T)],
                                   env={**os.environ, "GQ_DSTEP": ds}, capture_output=True, text=True, timeout=120)
                r.append(p.returncode)
            msg = ""
            if r == [0, 0]:
                import numpy as np
                a = np.load(f"/tmp/shape_1_{K}_{N}_{T}.npy"); b = np.load(f"/tmp/shape_0_{K}_{N}_{T}.npy")
                msg = f"err {np.max(np.abs(a-b))/np.max(np.abs(b)):.1e}"
            print(K, N, T, r, msg, flush=True)
