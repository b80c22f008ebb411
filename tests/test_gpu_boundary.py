"""The drop-in boundary from the reference's side (INTEGRATION.md route 1):

* the reference's OWN ``gridlq.pcg_solve`` (installed unmodified into ``baseline/_ref``)
  drives ``GpuSchurOperator`` / ``GpuNestedJacobiPreconditioner`` through its duck-typed
  contract (``pcg.py:53-60``; the template is ``NegatedOperator`` in
  ``tests/test_pcg.py:21-29``) and reproduces the golden runs;
* the device failure paths map onto the reference's exceptions: the pair-factor pivot rule
  (``block_linalg.py:54-60``, ``k_factor``'s SetupErr), a non-SPD cost block reaching the
  device directly through the C ABI (``k_spd_inverse``), and the device breakdown flag
  (``pcg.py:103-107``, reference test ``test_pcg.py:161-164``);
* unsupported state dimensions are refused with a clean error.
"""

import ctypes
import os
import sys

import numpy as np
import pytest

from conftest import load_golden, rel_err

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture(scope="module")
def gridlq():
    if not os.path.isdir(os.path.join(REF, "gridlq")):
        pytest.skip("reference not installed in baseline/_ref")
    sys.path.insert(0, REF)
    try:
        import gridlq as g
    finally:
        sys.path.remove(REF)
    return g


@pytest.mark.parametrize("name", ["config1", "config2", "boundary", "odd_kn", "time_varying",
                                  "cg"])
def test_reference_pcg_drives_gpu_operators(gridlq, name):
    from paper_2304_04980_b200 import GpuNestedJacobiPreconditioner, GpuSchurOperator

    ga, rec = load_golden(name)
    op = GpuSchurOperator(ga, rec["L"], rec["S"])
    pc = GpuNestedJacobiPreconditioner(op, rec["L"], rec["S"]) if rec["precond"] else None
    try:
        x, rep = gridlq.pcg_solve(op, pc, ga.offset, tol=rec["tol"], max_steps=rec["max_steps"])
    except gridlq.MaxIterationsExceeded as exc:
        x, rep = exc.iterate, exc.report
    assert rep.steps == int(rec["steps"])
    assert rel_err(x, rec["x"]) < 1e-9
    h, ho = np.array(rep.residual_inf_history), np.asarray(rec["hist"])
    assert np.all(np.abs(h - ho) <= 1e-9 * ho + 1e-14 * ho[0])
    # the reference's own flop bookkeeping over our counters (pcg.py:76-131)
    from paper_2304_04980_b200 import COUNT_KEYS
    got = np.array([rep.op_counts[k] for k in COUNT_KEYS])
    assert np.array_equal(got, rec["op_counts"])


def _ill_conditioned_pair_block():
    """config 1 with A = 1e10 I at node (0, 0): Psi's pair block there has a diagonal of
    ~1e20 next to O(1) pivots, below the reference's 1e-14 relative pivot rule."""
    ga, _ = load_golden("config1")
    A = ga.A.copy()
    A[0, 0, 0] = 1e10 * np.eye(ga.n)
    return ga.__class__(**{**ga.__dict__, "A": A})


def test_pair_factor_not_spd_on_device(gridlq):
    from paper_2304_04980_b200 import (GpuNestedJacobiPreconditioner, GpuSchurOperator,
                                       NotPositiveDefiniteError)
    from paper_2304_04980_b200.problem import arrays_to_problem

    bad = _ill_conditioned_pair_block()
    # the reference refuses it in its block-tridiagonal Cholesky (block_linalg.py:54-60)
    st = gridlq.build_stacked(arrays_to_problem(bad))
    with pytest.raises(gridlq.NotPositiveDefiniteError):
        gridlq.NestedJacobiPreconditioner(gridlq.build_schur(st), 2, 2)
    # ... and so does the device factorisation (k_factor's pivot test, gq_setup.cu)
    with pytest.raises(NotPositiveDefiniteError, match="pivot"):
        GpuNestedJacobiPreconditioner(GpuSchurOperator(bad, 2, 2), 2, 2)


def _create_raw(ga):
    """gq_create straight through the C ABI, without the host-side validation of
    ``GpuSchurOperator`` (the route a foreign caller of include/gridlq_b200.h takes)."""
    from paper_2304_04980_b200 import _lib

    keep = []

    def dptr(a):
        a = np.ascontiguousarray(a, dtype=np.float64)
        keep.append(a)
        return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))

    def iptr(a):
        a = np.ascontiguousarray(a, dtype=np.int32)
        keep.append(a)
        return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))

    desc = _lib.GqProblemDesc(
        K=ga.K, N=ga.N, T=ga.T, n=ga.n, m=ga.m, n_dyn=len(ga.A), n_cost=len(ga.Q),
        dyn_class=iptr(ga.dyn_class), cost_class=iptr(ga.cost_class),
        A=dptr(ga.A), B=dptr(ga.B), R=dptr(ga.R), C=dptr(ga.C), Q=dptr(ga.Q))
    lib = _lib.load()
    h = ctypes.c_void_p()
    rc = lib.gq_create(ctypes.byref(desc), 2, 2, ctypes.byref(h))
    if h.value:
        lib.gq_destroy(h)
    return rc, _lib.last_error(), h.value


def test_not_spd_cost_reaches_device_through_abi():
    """Q = -I handed straight to gq_create: the device Cholesky of the cost block
    (k_spd_inverse, same pivot rule as block_linalg.py:43-65) refuses it with GQ_NOT_SPD."""
    from paper_2304_04980_b200 import _lib

    ga, _ = load_golden("config1")
    bad = ga.__class__(**{**ga.__dict__,
                          "Q": -np.broadcast_to(np.eye(ga.n), ga.Q.shape).copy()})
    rc, msg, h = _create_raw(bad)
    assert rc == _lib.GQ_NOT_SPD, (rc, msg)
    assert h is None


def test_device_breakdown_flag(gridlq):
    """Curvature underflowing to zero (rhs scaled by 1e-170) stops the step on the device with
    the breakdown flag, as the reference's loop does (pcg.py:103-107)."""
    from paper_2304_04980_b200 import (BreakdownError, GpuNestedJacobiPreconditioner,
                                       GpuSchurOperator, pcg_solve)
    from paper_2304_04980_b200.problem import arrays_to_problem

    ga, _ = load_golden("config1")
    rhs = ga.offset * 1e-170
    st = gridlq.build_stacked(arrays_to_problem(ga))
    with pytest.raises(gridlq.BreakdownError):
        gridlq.pcg_solve(gridlq.build_schur(st),
                         gridlq.NestedJacobiPreconditioner(gridlq.build_schur(st), 2, 2), rhs,
                         tol=1e-320, max_steps=5)
    op = GpuSchurOperator(ga, 2, 2)
    with pytest.raises(BreakdownError):
        pcg_solve(op, GpuNestedJacobiPreconditioner(op, 2, 2), rhs, tol=1e-320, max_steps=5)


def test_unsupported_state_dimension():
    """n = 5 has no compiled kernel: refused on the host (DimensionMismatchError) and, through
    the raw C ABI, with GQ_UNSUPPORTED."""
    from paper_2304_04980_b200 import DimensionMismatchError, GpuSchurOperator, _lib
    from paper_2304_04980_b200 import generators

    ga = generators.random_case(4, 4, 3, 5, 1, seed=0)
    with pytest.raises(DimensionMismatchError):
        GpuSchurOperator(ga)
    rc, msg, h = _create_raw(ga)
    assert rc == _lib.GQ_UNSUPPORTED and "n=5" in msg, (rc, msg)
    assert h is None


def test_host_results_come_from_a_pinned_pool_without_aliasing():
    """Large host results live in page-locked memory from a pool: two results that are alive
    together never share a buffer, a view keeps its buffer out of the pool, and a dropped
    result's buffer is the next one handed out."""
    import gc

    from paper_2304_04980_b200 import (GpuNestedJacobiPreconditioner, GpuSchurOperator,
                                       MaxIterationsExceeded, generators, pcg_solve)
    from paper_2304_04980_b200.solver import _pinned

    ga = generators.msd_case(48, 40, 300, 0)          # 9.3 MB per vector: above the threshold
    op = GpuSchurOperator(ga, 2, 2)
    pc = GpuNestedJacobiPreconditioner(op, 2, 2)

    def solve(steps):
        try:
            return pcg_solve(op, pc, ga.offset, tol=1e-300, max_steps=steps)[0]
        except MaxIterationsExceeded as exc:
            return exc.iterate

    x3 = solve(3)
    if _pinned.take(4) is None:
        pytest.skip("page-locked host memory is not available")
    keep = x3.copy()
    x5 = solve(5)
    assert x3.ctypes.data != x5.ctypes.data
    assert np.array_equal(x3, keep)                   # the second solve did not touch it
    addr = x5.ctypes.data
    view = x5[10:20]
    vals = view.copy()
    del x5
    gc.collect()
    x4 = solve(4)                                     # x5's buffer is still held by the view
    assert x4.ctypes.data != addr and np.array_equal(view, vals)
    addr4 = x4.ctypes.data
    del x4
    gc.collect()
    x6 = solve(6)                                     # ... x4's came back and is re-used
    assert x6.ctypes.data == addr4
    assert np.array_equal(solve(3), keep)
