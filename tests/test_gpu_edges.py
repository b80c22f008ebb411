"""Edge shapes through the fast n = 2 / n = 4 kernels against the CPU oracle: single row or
column grids, odd sizes (padded pair blocks), a horizon of one stage, and T + 1 not a
multiple of the stencil / chain stage chunks.  20 PCG steps, iterates to 1e-9."""

import numpy as np
import pytest

from conftest import rel_err

pytestmark = pytest.mark.gpu

SHAPES = [
    (1, 1, 1, 2), (1, 5, 3, 2), (5, 1, 3, 2), (2, 3, 1, 2), (3, 2, 7, 2),
    (7, 9, 31, 2), (4, 6, 30, 2), (9, 4, 61, 2), (6, 5, 8, 4), (3, 3, 2, 4),
]


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("K,N,T,n", SHAPES)
def test_edge_shape_pcg(K, N, T, n):
    from oracle.gridlq_oracle import Oracle, pcg
    from paper_2304_04980_b200 import (GpuNestedJacobiPreconditioner, GpuSchurOperator,
                                       MaxIterationsExceeded, generators, pcg_solve)

    ga = generators.random_case(K, N, T, n, 1, seed=K * 100 + N * 10 + T, coupling_std=0.1)
    op = GpuSchurOperator(ga, 2, 2)
    pc = GpuNestedJacobiPreconditioner(op, 2, 2)
    orc = Oracle(ga, 2, 2)
    v = np.random.default_rng(0).standard_normal(op.dim)
    assert rel_err(op.apply(v), orc.apply_delta(v)) < 1e-12
    assert rel_err(pc.apply(v), orc.apply_precond(v)) < 1e-11
    steps = 20
    x_ref, hist_ref, k_ref, conv_ref, _ = pcg(orc, ga.offset, tol=1e-13, max_steps=steps)
    try:
        x, rep = pcg_solve(op, pc, ga.offset, tol=1e-13, max_steps=steps)
    except MaxIterationsExceeded as exc:
        x, rep = exc.iterate, exc.report
    assert rep.steps == k_ref
    assert rel_err(x, x_ref) < 1e-9
    h, hr = np.array(rep.residual_inf_history), np.array(hist_ref)
    assert np.all(np.abs(h - hr) <= 1e-9 * hr + 1e-14 * hr[0])


def test_n8_kernels_against_generic_multi_round():
    """n = 8 DMMA chain sweeps and block stencils against the generic thread-per-chain /
    per-node kernels on a size whose chain items take several persistent rounds (the
    SM-grouped item mapping must still cover every unit)."""
    import os
    import torch
    from paper_2304_04980_b200 import (GpuNestedJacobiPreconditioner, GpuSchurOperator,
                                       generators)

    ga = generators.config5(0, K=16, N=512, T=60)
    v = np.random.default_rng(3).standard_normal(ga.offset.shape[0])
    out = {}
    for tag, env in (("fast", {}), ("generic", {"GQ_NO_CHAIN": "1", "GQ_NO_ST8": "1"})):
        old = {k: os.environ.get(k) for k in ("GQ_NO_CHAIN", "GQ_NO_ST8")}
        os.environ.update(env)
        try:
            op = GpuSchurOperator(ga, 2, 2)
            pc = GpuNestedJacobiPreconditioner(op, 2, 2)
            out[tag] = (np.asarray(op.apply(v)), np.asarray(pc.apply(v)))
            del op, pc
            torch.cuda.empty_cache()
        finally:
            for k, val in old.items():
                if val is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = val
    assert rel_err(out["fast"][0], out["generic"][0]) < 1e-12
    assert rel_err(out["fast"][1], out["generic"][1]) < 1e-11


def test_solves_after_a_breakdown_on_a_padded_context():
    """Padded vector layout (T1 >= 60): a breakdown (curvature underflow) must not leave
    anything in the padding stages that reaches the flat reductions of the next solve -- plain
    CG afterwards (d.r and r.r over the padded span) reproduces the oracle."""
    from oracle.gridlq_oracle import Oracle, pcg
    from paper_2304_04980_b200 import (BreakdownError, GpuNestedJacobiPreconditioner,
                                       GpuSchurOperator, MaxIterationsExceeded, cg_solve,
                                       generators, pcg_solve)
    ga = generators.config2(0, K=6, N=6, T=63)
    op = GpuSchurOperator(ga, 2, 2)
    pc = GpuNestedJacobiPreconditioner(op, 2, 2)
    with pytest.raises(BreakdownError):
        pcg_solve(op, pc, ga.offset * 1e-170, tol=1e-320, max_steps=5)
    orc = Oracle(ga, 2, 2)
    xo, ho, so, _, _ = pcg(orc, ga.offset, tol=1e-30, max_steps=15, precond=False)
    try:
        x, rep = cg_solve(op, ga.offset, tol=1e-30, max_steps=15)
    except MaxIterationsExceeded as exc:
        x, rep = exc.iterate, exc.report
    h, ho = np.array(rep.residual_inf_history), np.array(ho)
    assert rep.steps == so == 15 and np.all(np.isfinite(h))
    assert np.all(np.abs(h - ho) <= 1e-9 * ho + 1e-14 * ho[0])
    assert np.max(np.abs(x - xo)) <= 1e-9 * np.max(np.abs(xo))
