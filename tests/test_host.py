"""Host-side logic (CPU only): ingestion, stage classes, flop counters, validation."""

import numpy as np
import pytest

import cases
from conftest import load_golden
from paper_2304_04980_b200 import generators as G
from paper_2304_04980_b200.counts import counters
from paper_2304_04980_b200.errors import DimensionMismatchError
from paper_2304_04980_b200.problem import (ConstSeq, GridLayout, arrays_from_problem,
                                           arrays_to_problem, validate_arrays)


def test_counters_match_reference(golden):
    name, ga, rec = golden
    c = counters(ga, rec["L"], rec["S"])
    for key in ("matvec_flops", "outer_coupling_flops", "inner_coupling_flops",
                "pair_solve_flops", "apply_flops"):
        assert c[key] == int(rec[key]), (name, key, c[key], int(rec[key]))


def test_roundtrip_problem_arrays():
    ga = G.config1(3)
    back = arrays_from_problem(arrays_to_problem(ga))
    for f in ("A", "B", "R", "C", "Q", "offset", "cmask", "dyn_class", "cost_class"):
        assert np.array_equal(getattr(back, f), getattr(ga, f)), f


def test_stage_classes_time_invariant():
    ga = G.config2(0)
    pc, pkeys = ga.psi_classes()
    xc, xkeys = ga.xi_classes()
    assert len(pkeys) == 2 and pc[0] == 0 and np.all(pc[1:] == 1)
    assert len(xkeys) == 1 and np.all(xc == 0)


def test_stage_classes_time_varying():
    ga = arrays_from_problem(cases.time_varying(T=5))
    pc, pkeys = ga.psi_classes()
    assert len(pkeys) == 6          # every stage distinct (terminal weight too)
    assert len(ga.xi_classes()[1]) == 5


def test_terminal_weight_class():
    p = arrays_to_problem(G.config1(0))
    T = p.T
    for row in p.subsystems:
        for s in row:
            q = list(s.Q)
            q[-1] = 2.0 * q[-1]
            s.Q = q
    ga = arrays_from_problem(p)
    assert list(ga.cost_class[:-1]) == [0] * T and ga.cost_class[-1] == 1
    pc, pkeys = ga.psi_classes()
    assert len(pkeys) == 3 and pc[-1] == 2


def test_heterogeneous_dimensions_rejected():
    p = cases.uncoupled(K=1, N=2, T=1)
    s = p.subsystems[0][1]
    s.n = 3
    s.A = [np.zeros((3, 3))]
    s.B = [np.zeros((3, 1))]
    s.Q = [np.eye(3)] * 2
    p.boundary.init[0][1] = np.ones(3)
    with pytest.raises(DimensionMismatchError):
        arrays_from_problem(p)


def test_invalid_problem_raises_value_error():
    p = arrays_to_problem(G.config1(0))
    s = p.subsystems[1][1]
    s.Q = ConstSeq(-np.eye(2), p.T + 1)
    with pytest.raises(ValueError, match="invalid problem"):
        arrays_from_problem(p)
    ga = G.config1(0)
    ga.R[0, 0, 0] = np.array([[0.0]])
    assert validate_arrays(ga)


def test_layout_matches_reference_order():
    lay = GridLayout(K=3, N=4, T=2, n=2)
    assert lay.x_offset(1, 2, 1) == 1 * 24 + (2 * 3 + 1) * 2
    assert lay.pairs == [(0, 1), (2, 3)]
    assert GridLayout(3, 5, 1, 1).pairs[-1] == (4,)


def test_boundary_offset_matches_reference():
    ga, rec = load_golden("boundary")
    assert np.array_equal(ga.offset, rec["ref_offset"])
    assert np.any(ga.offset[ga.K * ga.N * ga.n:] != 0)


def test_generators_are_seeded():
    a, b = G.config3(5, K=4, N=4, T=3), G.config3(5, K=4, N=4, T=3)
    assert np.array_equal(a.A, b.A) and np.array_equal(a.offset, b.offset)
    c = G.config3(6, K=4, N=4, T=3)
    assert not np.array_equal(a.A, c.A)
    m = G.config4(0, K=8, N=8, T=4)
    # spectral radius check of the MSD dynamics: stable-ish Euler discretisation
    assert m.n == 2 and m.m == 1 and np.all(np.isfinite(m.A))


def test_time_varying_ingestion_is_vectorised():
    """A time-varying GridLQProblem at 64 x 64 x 40 (every field per stage) converts in
    seconds: per-node sequences are stacked with one np.asarray each and equal stages found
    with one np.unique (problem._stage_ids), not a Python walk over T K N."""
    import time

    from paper_2304_04980_b200.problem import (BoundaryData, GridLQProblem, SubsystemData,
                                               arrays_from_problem)

    K = N = 64
    T, n, m = 40, 2, 1
    rng = np.random.default_rng(3)
    A = [0.3 * rng.standard_normal((n, n)) for _ in range(T)]
    A[7] = A[3]                                    # two stages share their dynamics
    B = [rng.standard_normal((n, m)) for _ in range(T)]
    B[7] = B[3]
    Q = [np.eye(n) * (1.0 + 0.01 * t) for t in range(T + 1)]
    R = [np.eye(m)] * T
    Cw = [0.01 * rng.standard_normal((n, n)) for _ in range(T)]
    Cw[7] = Cw[3]
    subs = []
    for i in range(K):
        row = []
        for j in range(N):
            kw = {d: Cw for d, ok in (("west", j > 0), ("east", j < N - 1), ("north", i > 0),
                                      ("south", i < K - 1)) if ok}
            row.append(SubsystemData(n=n, m=m, A=A, B=B, Q=Q, R=R, **kw))
        subs.append(row)
    init = [[np.ones(n) for _ in range(N)] for _ in range(K)]
    prob = GridLQProblem(K, N, T, subs, BoundaryData(init=init))
    t0 = time.perf_counter()
    ga = arrays_from_problem(prob)
    dt = time.perf_counter() - t0
    assert dt < 20.0, dt
    assert len(ga.A) == T - 1 and ga.dyn_class[7] == ga.dyn_class[3]
    assert len(ga.Q) == T + 1
    assert np.array_equal(ga.A[ga.dyn_class[5], 10, 20], A[5])


def _offset_from_boundary_arrays(problem, n):
    """numpy restatement of k_offset (csrc/gq_rhs.cu) on the arrays gq_build_offset receives."""
    from paper_2304_04980_b200.problem import boundary_arrays
    K, N, T = problem.K, problem.N, problem.T
    init, blk, cls, tr = boundary_arrays(problem, n)
    out = np.zeros((T + 1, N, K, n))
    out[0] = init
    for t in range(T):
        for j in range(N):
            for i in range(K):
                for d, edge, e in ((2, i == 0, j), (3, i == K - 1, j), (0, j == 0, i),
                                   (1, j == N - 1, i)):
                    if edge and cls[d, e, t] >= 0:
                        out[t + 1, j, i] += blk[d, e, cls[d, e, t]] @ tr[d, e, t]
    return out.reshape(-1)


def test_boundary_arrays_reproduce_reference_offset():
    """The dense inputs of the device omega~ kernel carry everything the reference's offset
    loop uses (kkt_assembly.py:275-301): all four edges, corners, missing trajectories."""
    p = cases.boundary_problem()
    _, rec = load_golden("boundary")
    assert np.allclose(_offset_from_boundary_arrays(p, 2), rec["ref_offset"], rtol=1e-15, atol=1e-16)
    p.boundary.south = None           # a direction without a trajectory contributes nothing
    from paper_2304_04980_b200.problem import rhs_offset
    assert np.allclose(_offset_from_boundary_arrays(p, 2), rhs_offset(p, 2), rtol=1e-15, atol=1e-16)
    tv = cases.time_varying()
    assert np.allclose(_offset_from_boundary_arrays(tv, 2), rhs_offset(tv, 2), rtol=1e-15, atol=1e-16)
