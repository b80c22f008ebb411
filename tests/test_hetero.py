"""Mixed subsystem dimensions (grid_problem.py:103-141) through the padded embedding
(paper_2304_04980_b200/embed.py).  CPU tier: index maps, the padded problem and the flop
counters against the reference's own numbers (tests/golden/hetero/hetero.npz, produced by
oracle/make_golden_hetero.py running the reference).  GPU tier: Delta, the preconditioner,
pcg_solve, primal recovery and the KKT residuals against the same fixture."""

import numpy as np
import pytest

import cases
from conftest import GOLDEN_DIR
from paper_2304_04980_b200.counts import counters
from paper_2304_04980_b200.embed import Embedding, is_heterogeneous
from paper_2304_04980_b200.problem import arrays_from_problem, rhs_offset

import os


def _golden():
    return np.load(os.path.join(GOLDEN_DIR, "hetero", "hetero.npz"), allow_pickle=False)


def test_embedding_maps_and_padded_offset():
    p = cases.hetero_problem()
    assert is_heterogeneous(p) and not is_heterogeneous(cases.boundary_problem())
    emb = Embedding(p)
    g = _golden()
    assert emb.dim == int(g["dim"]) and emb.n == 3 and emb.m == 2
    # expand / restrict are inverse on the real entries and pad with zeros
    v = np.arange(1, emb.dim + 1, dtype=float)
    big = emb.expand_x(v)
    assert big.shape == (emb.dim_pad,) and np.array_equal(emb.restrict_x(big), v)
    assert np.count_nonzero(big) == emb.dim
    with pytest.raises(Exception):
        emb.expand_x(np.zeros(emb.dim + 1))
    # the padded problem's omega~ restricted to the real entries is the reference's offset
    pp = emb.padded_problem(p)
    off = rhs_offset(pp, emb.n)
    assert np.allclose(emb.restrict_x(off), g["ref_offset"], rtol=1e-15, atol=1e-16)
    assert np.count_nonzero(off) == np.count_nonzero(g["ref_offset"])
    # layout slices follow the reference's GridLayout
    lay = emb.layout()
    assert lay.n_total == emb.dim and lay.x_slice(1, 2, 3).stop - lay.x_slice(1, 2, 3).start == \
        p.sub(1, 2).n


def test_counters_with_mixed_dimensions_match_reference():
    p = cases.hetero_problem()
    emb = Embedding(p)
    ga = arrays_from_problem(emb.padded_problem(p))
    c = counters(ga, 2, 2, nd=emb.nd)
    g = _golden()
    for k in ("matvec_flops", "outer_coupling_flops", "pair_solve_flops", "apply_flops"):
        assert c[k] == int(g[k]), k


@pytest.fixture(scope="module")
def gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.mark.gpu
def test_hetero_operator_preconditioner_and_pcg(gpu):
    from paper_2304_04980_b200 import (GpuNestedJacobiPreconditioner, GpuSchurOperator,
                                       kkt_residual, pcg_solve, recover_solution)
    g = _golden()
    p = cases.hetero_problem()
    op = GpuSchurOperator(p, 2, 2)
    pc = GpuNestedJacobiPreconditioner(op, 2, 2)
    assert op.dim == int(g["dim"])
    assert np.allclose(op.offset, g["ref_offset"], rtol=1e-15, atol=1e-16)
    assert np.allclose(op.offset_device().cpu().numpy(), g["ref_offset"], rtol=1e-15, atol=1e-16)
    v = g["v"]
    scale = np.max(np.abs(g["delta_v"]))
    assert np.max(np.abs(op.apply(v) - g["delta_v"])) <= 1e-12 * scale
    assert np.max(np.abs(op.apply_outer_coupling(v) - g["outer_v"])) <= 1e-12 * np.max(np.abs(g["outer_v"]))
    assert np.max(np.abs(pc.apply(v) - g["precond_v"])) <= 1e-11 * np.max(np.abs(g["precond_v"]))
    assert op.matvec_flops == int(g["matvec_flops"]) and pc.apply_flops == int(g["apply_flops"])
    x, rep = pcg_solve(op, pc, op.offset, tol=float(g["tol"]))
    h, href = np.array(rep.residual_inf_history), g["hist"]
    assert rep.steps == int(g["steps"]) and rep.converged
    assert np.all(np.abs(h - href) <= 1e-9 * href + 1e-14 * href[0])
    assert np.max(np.abs(x - g["x"])) <= 1e-9 * np.max(np.abs(g["x"]))
    ref_counts = dict(zip([str(k) for k in g["op_keys"]], g["op_vals"]))
    for k, val in rep.op_counts.items():
        assert val == ref_counts[k], k
    # device right-hand side and a CUDA-tensor solve give the same iterate
    xd, _ = pcg_solve(op, pc, op.offset_device(), tol=float(g["tol"]))
    assert np.allclose(xd.cpu().numpy(), x, rtol=1e-12, atol=1e-14)
    # recovery and KKT residuals in the reference's (unpadded) vector orders
    sol = recover_solution(op, x)
    assert sol.x_flat.shape == g["sol_x"].shape and sol.u_flat.shape == g["sol_u"].shape
    assert np.max(np.abs(sol.x_flat - g["sol_x"])) <= 1e-9 * np.max(np.abs(g["sol_x"]))
    assert np.max(np.abs(sol.u_flat - g["sol_u"])) <= 1e-9 * np.max(np.abs(g["sol_u"]))
    assert abs(sol.objective_value - float(g["objective"])) <= 1e-10 * abs(float(g["objective"]))
    assert sol.state(1, 2).shape == (p.T + 1, p.sub(1, 2).n)
    rx, ru, rdyn = kkt_residual(op, sol)
    assert rx <= 1e-12 and ru <= 1e-12 and rdyn <= 10 * float(g["kkt"][2]) + 1e-12


@pytest.mark.gpu
def test_uniform_dimension_without_compiled_kernels(gpu):
    """n = 5 has no compiled kernels; as a GridLQProblem it runs embedded in n = 8 and matches
    the numpy oracle (which restates the reference for any n) step for step."""
    from oracle.gridlq_oracle import Oracle, pcg
    from paper_2304_04980_b200 import (GpuNestedJacobiPreconditioner, GpuSchurOperator,
                                       MaxIterationsExceeded, generators, pcg_solve)
    from paper_2304_04980_b200.problem import arrays_to_problem
    ga = generators.random_case(4, 5, 3, 5, 2, seed=0)
    op = GpuSchurOperator(arrays_to_problem(ga), 2, 2)
    assert op.dim == ga.dim and op._embed.n == 8
    pc = GpuNestedJacobiPreconditioner(op, 2, 2)
    orc = Oracle(ga, 2, 2)
    v = np.random.default_rng(1).standard_normal(ga.dim)
    ref = orc.apply_delta(v)
    assert np.max(np.abs(op.apply(v) - ref)) <= 1e-12 * np.max(np.abs(ref))
    xo, ho, so, _, _ = pcg(orc, ga.offset, tol=1e-30, max_steps=12)
    try:
        x, rep = pcg_solve(op, pc, ga.offset, tol=1e-30, max_steps=12)
    except MaxIterationsExceeded as exc:
        x, rep = exc.iterate, exc.report
    h, ho = np.array(rep.residual_inf_history), np.array(ho)
    assert rep.steps == so == 12
    assert np.all(np.abs(h - ho) <= 1e-9 * ho + 1e-14 * ho[0])
    assert np.max(np.abs(x - xo)) <= 1e-9 * np.max(np.abs(xo))
