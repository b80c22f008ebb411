"""Parity of the B200 path (through the C-ABI) against golden vectors from the reference
and against the CPU oracle.  Needs a CUDA device: ``pytest -m gpu``."""

import numpy as np
import pytest

from conftest import history_ok, load_golden, rel_err
from test_oracle_golden import CHAOTIC_PREFIX, check_run

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _ops(ga, rec):
    from paper_2304_04980_b200 import GpuNestedJacobiPreconditioner, GpuSchurOperator

    op = GpuSchurOperator(ga, rec["L"], rec["S"])
    pc = GpuNestedJacobiPreconditioner(op, rec["L"], rec["S"])
    return op, pc


def test_unit_applies(golden):
    name, ga, rec = golden
    op, pc = _ops(ga, rec)
    v = rec["vec"]
    assert rel_err(op.apply(v), rec["delta"]) < 1e-12
    assert rel_err(op.apply_outer_coupling(v), rec["outer"]) < 1e-12
    assert rel_err(pc.apply_inner_coupling(v), rec["inner"]) < 1e-12
    assert rel_err(pc.pair_solves(v), rec["pair"]) < 1e-11
    if "prec" in rec:
        assert rel_err(pc.apply(v), rec["prec"]) < 1e-11


def _solve(ga, rec, callback=None):
    from paper_2304_04980_b200 import MaxIterationsExceeded, pcg_solve

    op, pc = _ops(ga, rec)
    try:
        x, rep = pcg_solve(op, pc if rec["precond"] else None, ga.offset, tol=rec["tol"],
                           max_steps=rec["max_steps"], x0=rec.get("x0"), callback=callback)
    except MaxIterationsExceeded as exc:
        x, rep = exc.iterate, exc.report
        assert exc.iterations == rep.steps
    return op, pc, x, rep


def test_pcg_parity(golden):
    name, ga, rec = golden
    snaps = {}

    def cb(step, x, r):
        if step in set(int(s) for s in rec["snap_steps"]):
            snaps[step] = x.copy()

    op, pc, x, rep = _solve(ga, rec)
    check_run(name, rec, x, rep.residual_inf_history, rep.steps, rep.converged,
              {int(s): xs for s, xs in zip(rec["snap_steps"], rec["snap_x"])})
    # op_counts bookkeeping identical to the reference (pcg.py:76-131)
    if name not in CHAOTIC_PREFIX:
        from paper_2304_04980_b200 import COUNT_KEYS
        got = np.array([rep.op_counts[k] for k in COUNT_KEYS])
        assert np.array_equal(got, rec["op_counts"]), (got, rec["op_counts"])
    # intermediate iterates through the callback path
    if len(rec["snap_steps"]) and max(rec["snap_steps"]) <= 60:
        _, _, x2, rep2 = _solve(ga, rec, callback=cb)
        for s, xs in zip(rec["snap_steps"], rec["snap_x"]):
            if name not in CHAOTIC_PREFIX or s <= CHAOTIC_PREFIX[name]:
                assert rel_err(snaps[int(s)], xs) < 1e-9
        assert np.array_equal(x2, x)   # bitwise run-to-run reproducibility


def test_device_pointer_roundtrip():
    import torch

    from paper_2304_04980_b200 import GpuSchurOperator

    ga, rec = load_golden("config1")
    op = GpuSchurOperator(ga)
    v = torch.tensor(rec["vec"], device="cuda", dtype=torch.float64)
    y = op.apply(v)
    assert y.is_cuda
    assert rel_err(y.cpu().numpy(), rec["delta"]) < 1e-12


def test_failure_modes():
    from paper_2304_04980_b200 import (DimensionMismatchError, GpuNestedJacobiPreconditioner,
                                       GpuSchurOperator, MaxIterationsExceeded, cg_solve,
                                       pcg_solve)

    ga, rec = load_golden("msd_ref")
    op = GpuSchurOperator(ga)
    pc = GpuNestedJacobiPreconditioner(op, 2, 2)
    with pytest.raises(MaxIterationsExceeded) as info:
        pcg_solve(op, pc, ga.offset, tol=1e-9, max_steps=2)
    exc = info.value
    assert exc.iterations == 2 and exc.report is not None and not exc.report.converged
    assert exc.iterate.shape == (op.dim,)
    with pytest.raises(DimensionMismatchError):
        cg_solve(op, np.zeros(op.dim + 1))
    with pytest.raises(ValueError):
        cg_solve(op, np.full(op.dim, np.nan))
    with pytest.raises(ValueError):
        cg_solve(op, ga.offset, tol=0.0)
    with pytest.raises(ValueError, match="even"):
        GpuNestedJacobiPreconditioner(op, 1, 2).apply(np.zeros(op.dim))
    with pytest.raises(ValueError):
        GpuNestedJacobiPreconditioner(op, 0, 2)


def test_not_spd_problem_rejected():
    from paper_2304_04980_b200 import GpuSchurOperator

    ga, _ = load_golden("config1")
    bad = ga.__class__(**{**ga.__dict__, "Q": -ga.Q})
    with pytest.raises(ValueError, match="invalid problem"):
        GpuSchurOperator(bad)


def test_identity_operator_one_step():
    """Delta = I (uncoupled, A = 0, B = 0): CG converges in one step (test_pcg.py:43-50)."""
    from paper_2304_04980_b200 import GpuSchurOperator, cg_solve

    ga, _ = load_golden("uncoupled")
    op = GpuSchurOperator(ga)
    rhs = np.random.default_rng(0).standard_normal(op.dim)
    x, rep = cg_solve(op, rhs, tol=1e-9)
    assert rep.steps == 1 and rep.converged
    assert np.max(np.abs(x - rhs)) < 1e-12


# ---- full-size checks at the BASELINE configurations ------------------------------------

@pytest.mark.parametrize("cfg", [4, 3])
def test_full_size_operator_parity(cfg):
    """Delta and the preconditioner at the BASELINE sizes against the CPU oracle."""
    from oracle.gridlq_oracle import Oracle
    from paper_2304_04980_b200 import (GpuNestedJacobiPreconditioner, GpuSchurOperator,
                                       generators)

    ga = generators.CONFIGS[cfg](0)
    S = 3 if cfg == 3 else 2
    op = GpuSchurOperator(ga, 2, S)
    pc = GpuNestedJacobiPreconditioner(op, 2, S)
    orc = Oracle(ga, 2, S)
    v = np.random.default_rng(1).standard_normal(op.dim)
    assert rel_err(op.apply(v), orc.apply_delta(v)) < 1e-12
    assert rel_err(pc.apply(v), orc.apply_precond(v)) < 1e-11


def test_headline_properties():
    """Size-independent properties at K=N=256, T=200: symmetry of Delta and of the
    preconditioner, linearity, and 100 PCG steps whose recurred residual tracks the true
    residual (test_pcg.py:117-129) with a decreasing history."""
    import torch

    from paper_2304_04980_b200 import (GpuNestedJacobiPreconditioner, GpuSchurOperator,
                                       MaxIterationsExceeded, generators, pcg_solve)

    ga = generators.config4(0)
    op = GpuSchurOperator(ga)
    pc = GpuNestedJacobiPreconditioner(op, 2, 2)
    g = torch.Generator(device="cuda").manual_seed(0)
    a = torch.randn(op.dim, device="cuda", dtype=torch.float64, generator=g)
    b = torch.randn(op.dim, device="cuda", dtype=torch.float64, generator=g)
    da, db = op.apply(a), op.apply(b)
    s1, s2 = float(torch.dot(da, b)), float(torch.dot(a, db))
    assert abs(s1 - s2) < 1e-10 * max(abs(s1), 1.0)
    pa, pb = pc.apply(a), pc.apply(b)
    s1, s2 = float(torch.dot(pa, b)), float(torch.dot(a, pb))
    assert abs(s1 - s2) < 1e-10 * max(abs(s1), 1.0)
    pab = pc.apply(a + b)
    assert float((pab - pa - pb).abs().max()) < 1e-12 * float(pab.abs().max())
    assert float(torch.dot(pa, a)) > 0
    rhs = torch.tensor(ga.offset, device="cuda")
    with pytest.raises(MaxIterationsExceeded) as info:
        pcg_solve(op, pc, rhs, tol=1e-30, max_steps=100)
    rep = info.value.report
    x = info.value.iterate
    h = np.array(rep.residual_inf_history)
    assert rep.steps == 100 and h[-1] < 1e-6 * h[0]
    true_r = rhs - op.apply(x)
    assert float(true_r.abs().max()) < 1e-8 * float(rhs.abs().max()) + 10 * h[-1]


def test_nbjm_parity(nbjm_golden):
    """Device standalone nested Jacobi solve vs the reference's nbjm_solve."""
    from paper_2304_04980_b200 import (GpuNestedJacobiPreconditioner, GpuSchurOperator,
                                       MaxIterationsExceeded, nbjm_solve)

    name, ga, rec = nbjm_golden
    op = GpuSchurOperator(ga, rec["L"], 1)
    pc = GpuNestedJacobiPreconditioner(op, rec["L"], 1)
    if rec["converged"]:
        x, outers = nbjm_solve(pc, ga.offset, tol=rec["tol"], max_outer=rec["max_outer"])
    else:
        with pytest.raises(MaxIterationsExceeded) as info:
            pc.solve(ga.offset, tol=rec["tol"], max_outer=rec["max_outer"])
        x, outers = info.value.iterate, info.value.iterations
        assert x is not None
    assert outers == rec["outers"]
    assert rel_err(x, rec["x"]) < 1e-9
    # the fixed point solves Delta x = rhs
    if rec["converged"]:
        res = np.max(np.abs(op.apply(x) - ga.offset)) / np.max(np.abs(ga.offset))
        assert res < 1e-6


def test_nbjm_budget_and_device_vectors():
    """max_outer < 1 raises with no iterate (the reference loop never runs); torch device
    vectors in and out."""
    import torch
    from paper_2304_04980_b200 import (GpuNestedJacobiPreconditioner, GpuSchurOperator,
                                       MaxIterationsExceeded, generators)

    ga = generators.config1(0)
    op = GpuSchurOperator(ga, 2, 2)
    pc = GpuNestedJacobiPreconditioner(op, 2, 2)
    with pytest.raises(MaxIterationsExceeded) as info:
        pc.solve(ga.offset, max_outer=0)
    assert info.value.iterate is None
    rhs = torch.tensor(ga.offset, device="cuda", dtype=torch.float64)
    with pytest.raises(MaxIterationsExceeded) as info:
        pc.solve(rhs, tol=1e-30, max_outer=4)
    assert isinstance(info.value.iterate, torch.Tensor) and info.value.iterations == 4
    with pytest.raises(MaxIterationsExceeded) as info2:
        pc.solve(ga.offset, tol=1e-30, max_outer=4)
    assert rel_err(info.value.iterate.cpu().numpy(), info2.value.iterate) < 1e-15


@pytest.mark.parametrize("case", ["n8", "n4", "n1_oddk"])
def test_nbjm_vs_oracle_other_block_sizes(case):
    """Standalone nested Jacobi on the n = 8 (DMMA chain + k_st8), n = 4 and n = 1 paths
    against the oracle restatement (outer-sweep count and solution)."""
    from oracle.gridlq_oracle import Oracle
    from paper_2304_04980_b200 import (GpuNestedJacobiPreconditioner, GpuSchurOperator,
                                       generators)

    if case == "n8":
        ga = generators.config5(0, K=4, N=6, T=3)
    elif case == "n4":
        ga = generators.config3(0, K=4, N=4, T=4)
    else:
        ga = generators.random_case(5, 3, 4, 1, 1, seed=5)
    op = GpuSchurOperator(ga, 2, 1)
    pc = GpuNestedJacobiPreconditioner(op, 2, 1)
    tol = 1e-9 * float(np.max(np.abs(ga.offset)))
    xo, no, conv = Oracle(ga, 2, 1).nbjm_solve(ga.offset, tol=tol, max_outer=3000)
    assert conv
    x, n = pc.solve(ga.offset, tol=tol, max_outer=3000)
    assert n == no
    assert rel_err(x, xo) < 1e-9
