"""Pin the CPU oracle against golden vectors produced by the reference itself
(``oracle/make_golden.py``).  CPU only."""

import numpy as np
import pytest

from conftest import history_ok, rel_err
from oracle.gridlq_oracle import Oracle, pcg

# the largest fixtures take a few seconds of oracle PCG each
HEAVY = {"config2", "config4r", "config3r"}
# Unpreconditioned CG on the reference's planar MSD case amplifies rounding so fast that
# ANY reordering of the reductions (even inside the reference) drifts O(1) after ~40
# steps; compare its history on the well-conditioned prefix and the converged solution.
CHAOTIC_PREFIX = {"msd_ref_cg": 20}


def test_offset_and_operators(golden):
    name, ga, rec = golden
    assert np.array_equal(ga.offset, rec["ref_offset"])
    orc = Oracle(ga, rec["L"], rec["S"])
    v = rec["vec"]
    assert rel_err(orc.apply_delta(v), rec["delta"]) < 1e-13
    assert rel_err(orc.apply_outer(v), rec["outer"]) < 1e-13
    assert rel_err(orc.apply_inner(v), rec["inner"]) < 1e-13
    assert rel_err(orc.pair_solve(v), rec["pair"]) < 1e-12
    if "prec" in rec:
        assert rel_err(orc.apply_precond(v), rec["prec"]) < 1e-12


def test_pcg_parity(golden):
    name, ga, rec = golden
    if name in HEAVY:
        pytest.skip("covered by the GPU parity suite; oracle PCG too slow for the CPU tier")
    orc = Oracle(ga, rec["L"], rec["S"])
    snaps = {}

    def cb(step, x, r):
        snaps[step] = x.copy()

    x, hist, steps, conv, status = pcg(orc, ga.offset, tol=rec["tol"], max_steps=rec["max_steps"],
                                       x0=rec.get("x0"), precond=bool(rec["precond"]),
                                       callback=cb)
    check_run(name, rec, x, hist, steps, conv, snaps)


def check_run(name, rec, x, hist, steps, conv, snaps):
    """Parity rule shared by the oracle and GPU suites."""
    prefix = CHAOTIC_PREFIX.get(name)
    if prefix is None:
        assert history_ok(hist, rec["hist"])
        assert steps == int(rec["steps"]) and int(conv) == int(rec["converged"])
        assert rel_err(x, rec["x"]) < 1e-9
    else:
        assert history_ok(list(hist)[:prefix], rec["hist"][:prefix])
        assert int(conv) == int(rec["converged"])
        assert rel_err(x, rec["x"]) < 1e-6
    for s, xs in zip(rec["snap_steps"], rec["snap_x"]):
        if (prefix is None or s <= prefix) and int(s) in snaps:
            assert rel_err(snaps[int(s)], xs) < 1e-9


def test_odd_inner_budget_refused():
    from conftest import load_golden

    ga, _ = load_golden("config1")
    orc = Oracle(ga, 3, 3)
    with pytest.raises(ValueError, match="even"):
        orc.apply_precond(np.zeros(orc.dim))


def test_c_oracle_matches_golden(golden):
    """The C restatement (CPU baseline) against the reference's golden vectors."""
    from oracle.coracle import COracle

    name, ga, rec = golden
    co = COracle(Oracle(ga, rec["L"], rec["S"]))
    v = rec["vec"]
    assert rel_err(co.apply_delta(v), rec["delta"]) < 1e-13
    assert rel_err(co.apply_outer(v), rec["outer"]) < 1e-13
    assert rel_err(co.apply_inner(v), rec["inner"]) < 1e-13
    assert rel_err(co.pair_solve(v), rec["pair"]) < 1e-12
    if "prec" in rec:
        assert rel_err(co.apply_precond(v), rec["prec"]) < 1e-12
    if rec.get("x0") is None:
        x, hist, steps, conv, status, _ = co.pcg(ga.offset, tol=rec["tol"],
                                                 max_steps=rec["max_steps"],
                                                 precond=bool(rec["precond"]))
        check_run(name, rec, x, hist, steps, conv, {})


def test_nbjm_parity(nbjm_golden):
    """Standalone nested Jacobi (nested_jacobi.py:124-151): same outer-sweep count and the
    same solution / last iterate as the reference."""
    name, ga, rec = nbjm_golden
    assert np.array_equal(ga.offset, rec["ref_offset"])
    orc = Oracle(ga, rec["L"], 1)
    x, outers, conv = orc.nbjm_solve(ga.offset, tol=rec["tol"], max_outer=rec["max_outer"])
    assert int(conv) == rec["converged"]
    assert outers == rec["outers"]
    assert rel_err(x, rec["x"]) < 1e-9
