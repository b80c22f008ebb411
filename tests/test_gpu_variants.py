"""Every kernel variant the library can select stays parity-green: the golden unit-apply and
PCG parity tests re-run in a subprocess per variant (the selections are read from the
environment when a context is created or a kernel is launched)."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))

VARIANTS = {
    "generic_v1": {"GQ_FORCE_V1": "1"},          # thread-per-chain sweeps, v1 stencils
    "no_chain": {"GQ_NO_CHAIN": "1"},            # FMA / v6 sweeps instead of the chain kernel
    "no_grid": {"GQ_NO_GRID": "1"},              # v2 stencils instead of the n=2 grid kernel
    "chainm": {"GQ_CHAINM": "2"},                # twelve-warp chain sweeps (every form) on the n=2 cases
    "dstep": {"GQ_DSTEP": "1"},                  # t-loop Delta + tiled outer rhs on every (small) golden case
    "dstep_no_rstep": {"GQ_DSTEP": "1", "GQ_NO_RSTEP": "1"},   # ... with the lane-per-stage outer rhs
    "fuse_x": {"GQ_FUSE_X": "1"},                # x update fused into the direction update
    "no_fuse_x": {"GQ_FUSE_X": "0"},             # ... and on its own graph branch for small sizes
    "no_fuse_r": {"GQ_NO_FUSE_R": "1"},          # separate r update kernel
    "no_fuse": {"GQ_NO_FUSE_R": "1", "GQ_NO_FORK": "1"},
    "no_fork": {"GQ_NO_FORK": "1"},              # x update in line instead of on a branch
}


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("variant", sorted(VARIANTS))
def test_variant_parity(variant):
    env = dict(os.environ, **VARIANTS[variant])
    cmd = [sys.executable, "-m", "pytest", os.path.join(HERE, "test_gpu_parity.py"), "-q", "-x",
           "-m", "gpu", "-k", "unit_applies or pcg_parity or not_spd or nbjm", "-p", "no:cacheprovider"]
    res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-2000:]
