"""Device-side right-hand side omega~ (gq_build_offset, csrc/gq_rhs.cu) against the
reference's offset loop (kkt_assembly.py:275-301): the golden boundary case (offset produced
by the reference itself), a time-varying problem, a direction without a trajectory, and the
headline size through pcg_solve with the right-hand side never leaving the device."""

import numpy as np
import pytest

import cases
from conftest import load_golden
from paper_2304_04980_b200 import (ConstSeq, GpuNestedJacobiPreconditioner, GpuSchurOperator,
                                   MaxIterationsExceeded, generators, pcg_solve,
                                   rhs_offset_device)
from paper_2304_04980_b200.problem import arrays_to_problem, rhs_offset

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_device_offset_matches_reference_golden():
    p = cases.boundary_problem()
    _, rec = load_golden("boundary")
    off = rhs_offset_device(p).cpu().numpy()
    assert np.allclose(off, rec["ref_offset"], rtol=1e-15, atol=1e-16)
    assert np.any(off[p.K * p.N * 2:] != 0)


def test_device_offset_time_varying_and_missing_direction():
    tv = cases.time_varying()
    assert np.allclose(rhs_offset_device(tv).cpu().numpy(), rhs_offset(tv, 2), rtol=1e-15,
                       atol=1e-16)
    p = cases.boundary_problem(K=4, N=5, T=6, seed=3)
    p.boundary.west = None
    assert np.allclose(rhs_offset_device(p).cpu().numpy(), rhs_offset(p, 2), rtol=1e-15,
                       atol=1e-16)
    # per-stage coupling blocks on one edge node (a plain list, not a ConstSeq)
    rng = np.random.default_rng(5)
    p.subsystems[0][2].north = [0.05 * rng.standard_normal((2, 2)) for _ in range(p.T)]
    assert np.allclose(rhs_offset_device(p).cpu().numpy(), rhs_offset(p, 2), rtol=1e-15,
                       atol=1e-16)


def test_operator_offset_device_feeds_pcg():
    """build_schur from a GridLQProblem: omega~ is built on the device and drives pcg_solve."""
    p = cases.boundary_problem(K=6, N=6, T=8, seed=9)
    op = GpuSchurOperator(p, 2, 2)
    pc = GpuNestedJacobiPreconditioner(op, 2, 2)
    rhs = op.offset_device()
    assert rhs.is_cuda and np.allclose(rhs.cpu().numpy(), op.offset, rtol=1e-15, atol=1e-16)
    x_dev, rep_dev = pcg_solve(op, pc, rhs, tol=1e-10)
    x_host, rep_host = pcg_solve(op, pc, op.offset, tol=1e-10)
    assert rep_dev.steps == rep_host.steps
    assert np.allclose(x_dev.cpu().numpy(), x_host, rtol=1e-9, atol=1e-12)


def test_device_offset_headline_size():
    """K = N = 256, T = 200: omega~ = [x0; 0] from the device kernel equals the generator's."""
    ga = generators.config4(0)
    p = arrays_to_problem(ga)
    off = rhs_offset_device(p)
    assert off.numel() == ga.dim
    assert np.array_equal(off.cpu().numpy(), ga.offset)
