"""Full-size PCGM parity against the pinned C oracle (north_star: iterates, residual history
and final solution within 1e-9 relative after the same fixed number of steps; the same
iteration count to a tolerance).

The oracle is ``oracle/gridlq_oracle.c`` (restating ``pcg.py:98-131`` over the numpy
oracle's setup, pinned to the reference's own outputs by ``test_oracle_golden.py``), run
on all host threads.  The reference itself cannot hold these sizes.

* config 4 (the headline, K = N = 256, T = 200, S = L = 2): 100 fixed steps;
* config 3 (K = N = 64, T = 100, n = 4) with S = 3 and L in {2, 4} (L = 3 is refused by the
  reference): 200 fixed steps -- far past convergence, so the history is
  compared with the 1e-14 h0 floor of SURVEY.md 8(c);
* config 5 (n = 8, m = 4, S = L = 2) to 1e-10 ||omega~||_inf on K = 32, N = 256, T = 500
  (a quarter of the BASELINE grid, as VERDICT r1 asks when the full size is out of reach
  of the CPU oracle's step time): equal step counts and final iterates.
"""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _solve_both(ga, S, L, tol, max_steps):
    from oracle.coracle import COracle
    from oracle.gridlq_oracle import Oracle
    from paper_2304_04980_b200 import (GpuNestedJacobiPreconditioner, GpuSchurOperator,
                                       MaxIterationsExceeded, pcg_solve)

    orc = COracle(Oracle(ga, L, S), threads=os.cpu_count())
    xo, ho, ko, convo, _, _ = orc.pcg(ga.offset, tol=tol, max_steps=max_steps)
    op = GpuSchurOperator(ga, L, S)
    pc = GpuNestedJacobiPreconditioner(op, L, S)
    try:
        x, rep = pcg_solve(op, pc, ga.offset, tol=tol, max_steps=max_steps)
    except MaxIterationsExceeded as exc:
        x, rep = exc.iterate, exc.report
    return (np.asarray(x), np.array(rep.residual_inf_history), rep.steps, rep.converged,
            xo, np.array(ho), ko, convo)


def _check(res, hist_all=True):
    x, h, k, conv, xo, ho, ko, convo = res
    assert k == ko and conv == convo, (k, ko, conv, convo)
    err = np.max(np.abs(x - xo)) / np.max(np.abs(xo))
    assert err < 1e-9, f"iterate rel err {err:.3e}"
    # |h - h_ref| <= 1e-9 h_ref + 1e-14 h_0
    bad = np.abs(h - ho) > 1e-9 * ho + 1e-14 * ho[0]
    assert not bad.any(), f"history mismatch at steps {np.nonzero(bad)[0][:5]}"
    return err


def test_headline_100_fixed_steps():
    from paper_2304_04980_b200 import generators

    ga = generators.config4(0)
    res = _solve_both(ga, 2, 2, 1e-300, 100)
    assert res[2] == 100
    _check(res)


@pytest.mark.parametrize("shape", [(16, 512, 200), (33, 255, 171)])
def test_wide_grids_many_rounds_of_the_twelve_warp_kernel(shape):
    """Grids whose chain items need more than two rounds of the twelve-warp kernel (6656 items
    at 16 x 512 x 200: four rounds), and odd K / N / chunk counts with a partial last round
    and a short last chunk, against the C oracle: 40 fixed steps."""
    from paper_2304_04980_b200 import generators

    K, N, T = shape
    ga = generators.config4(3, K=K, N=N, T=T)
    res = _solve_both(ga, 2, 2, 1e-300, 40)
    assert res[2] == 40
    _check(res)


@pytest.mark.parametrize("L", [2, 4])
def test_config3_200_fixed_steps(L):
    from paper_2304_04980_b200 import generators

    ga = generators.config3(0)
    res = _solve_both(ga, 3, L, 1e-300, 200)
    assert res[2] == 200
    _check(res)


def test_config5_to_tolerance():
    from paper_2304_04980_b200 import generators

    ga = generators.config5(0, K=32, N=256, T=500)
    tol = 1e-10 * float(np.max(np.abs(ga.offset)))
    res = _solve_both(ga, 2, 2, tol, 2000)
    assert res[3] and res[7], "both solves reach the tolerance"
    _check(res)


@pytest.mark.skipif(os.environ.get("GQ_FULL_C5") != "1",
                    reason="full-size config 5 (~8 min of CPU oracle): GQ_FULL_C5=1")
def test_config5_full_size_to_tolerance():
    """The BASELINE grid itself (K = 32, N = 1024, T = 500, dim 131M); the oracle needs about
    12 GB of host memory and minutes of 16-thread step time."""
    from paper_2304_04980_b200 import generators

    ga = generators.config5(0)
    tol = 1e-10 * float(np.max(np.abs(ga.offset)))
    res = _solve_both(ga, 2, 2, tol, 2000)
    assert res[3] and res[7], "both solves reach the tolerance"
    err = _check(res)
    print(f"config 5 full size: {res[2]} steps on both, max rel iterate err {err:.2e}")
