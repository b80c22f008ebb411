"""The TMA-tile kernels (t-loop Delta `k_dstep`, outer rhs `k_rstep`) on shapes that hit their
tile and chunk boundaries, forced on small grids with GQ_DSTEP=1 and checked against the CPU
oracle: grids that overhang the 16 x 8 / 32 x 8 tiles, horizons of one and two stages (the
outer rhs needs T >= 2 and falls back below that), T a multiple of the 8-stage chunk, one more
and one less, and grids small enough that a tile's chunks are cut into pieces (items that start
inside a tile).  20 PCG steps, iterates to 1e-9."""

import numpy as np
import pytest

from conftest import rel_err

pytestmark = pytest.mark.gpu

SHAPES = [
    (17, 9, 1), (17, 9, 2), (16, 8, 8), (18, 10, 9), (33, 17, 16), (5, 3, 17), (20, 12, 25),
    (3, 20, 7), (40, 5, 33),
]


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


CASES = [(K, N, T, None) for K, N, T in SHAPES] + [
    (K, N, T, p) for K, N, T in [(17, 9, 2), (33, 17, 16), (20, 12, 25)] for p in ("1", "3")]


@pytest.mark.parametrize("K,N,T,pieces", CASES)
def test_tile_kernels_against_oracle(K, N, T, pieces, monkeypatch):
    from oracle.gridlq_oracle import Oracle, pcg
    from paper_2304_04980_b200 import (GpuNestedJacobiPreconditioner, GpuSchurOperator,
                                       MaxIterationsExceeded, generators, pcg_solve)

    monkeypatch.setenv("GQ_DSTEP", "1")
    if pieces is not None:
        monkeypatch.setenv("GQ_RS_PIECES", pieces)
    ga = generators.random_case(K, N, T, 2, 1, seed=K * 100 + N * 10 + T, coupling_std=0.1)
    op = GpuSchurOperator(ga, 2, 2)
    pc = GpuNestedJacobiPreconditioner(op, 2, 2)
    orc = Oracle(ga, 2, 2)
    v = np.random.default_rng(1).standard_normal(op.dim)
    assert rel_err(op.apply(v), orc.apply_delta(v)) < 1e-12
    assert rel_err(op.apply_outer_coupling(v), orc.apply_outer(v)) < 1e-12
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
