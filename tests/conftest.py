import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)

GOLDEN_DIR = os.path.join(HERE, "golden")
GOLDEN_CASES = sorted(os.path.splitext(os.path.basename(p))[0]
                      for p in glob.glob(os.path.join(GOLDEN_DIR, "*.npz"))
                      if not os.path.basename(p).startswith("nbjm_"))
# standalone nested Jacobi solves (nested_jacobi.py:124-151) run by the reference
NBJM_CASES = sorted(os.path.splitext(os.path.basename(p))[0]
                    for p in glob.glob(os.path.join(GOLDEN_DIR, "nbjm_*.npz")))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    """Golden record -> (GridArrays, dict of expected values)."""
    from paper_2304_04980_b200.problem import GridArrays

    z = np.load(os.path.join(GOLDEN_DIR, f"{name}.npz"))
    rec = {k: z[k] for k in z.files}
    ga = GridArrays(
        K=int(rec["K"]), N=int(rec["N"]), T=int(rec["T"]), n=int(rec["n"]), m=int(rec["m"]),
        A=rec["A"], B=rec["B"], R=rec["R"], C=rec["C"], cmask=rec["cmask"], Q=rec["Q"],
        dyn_class=rec["dyn_class"].astype(np.int32), cost_class=rec["cost_class"].astype(np.int32),
        offset=rec["offset"])
    rec["tol"] = float(rec["tol"])
    rec["L"] = int(rec["L"])
    rec["S"] = int(rec["S"])
    rec["max_steps"] = None if int(rec["max_steps"]) < 0 else int(rec["max_steps"])
    rec["status"] = str(rec["status"])
    return ga, rec


def load_nbjm(name):
    """NBJM golden record -> (GridArrays, dict: L, tol, max_outer, x, outers, converged)."""
    from paper_2304_04980_b200.problem import GridArrays

    z = np.load(os.path.join(GOLDEN_DIR, f"{name}.npz"))
    rec = {k: z[k] for k in z.files}
    ga = GridArrays(
        K=int(rec["K"]), N=int(rec["N"]), T=int(rec["T"]), n=int(rec["n"]), m=int(rec["m"]),
        A=rec["A"], B=rec["B"], R=rec["R"], C=rec["C"], cmask=rec["cmask"], Q=rec["Q"],
        dyn_class=rec["dyn_class"].astype(np.int32), cost_class=rec["cost_class"].astype(np.int32),
        offset=rec["offset"])
    for k in ("L", "max_outer", "outers", "converged"):
        rec[k] = int(rec[k])
    rec["tol"] = float(rec["tol"])
    return ga, rec


def rel_err(a, b):
    scale = max(float(np.max(np.abs(b))), 1e-300) if np.size(b) else 1.0
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b)))) / scale if np.size(b) else 0.0


def history_ok(h, ref, rtol=1e-9, floor=1e-14):
    """SURVEY.md 8(c) history rule: |h - ref| <= rtol*ref + floor*ref[0]."""
    h = np.asarray(h)
    ref = np.asarray(ref)
    if h.shape != ref.shape:
        return False
    return bool(np.all(np.abs(h - ref) <= rtol * ref + floor * ref[0]))


@pytest.fixture(params=GOLDEN_CASES)
def golden(request):
    return request.param, *load_golden(request.param)


@pytest.fixture(params=NBJM_CASES)
def nbjm_golden(request):
    return request.param, *load_nbjm(request.param)
