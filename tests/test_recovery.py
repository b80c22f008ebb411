"""Primal recovery and KKT residuals (recovery.py:50-80): the numpy oracle against the
reference's own outputs (golden vectors), and the B200 path against both."""

import numpy as np
import pytest

from conftest import GOLDEN_CASES as GOLDEN_NAMES
from conftest import load_golden, rel_err


def _oracle_check(name):
    from oracle.gridlq_oracle import kkt, recover

    ga, rec = load_golden(name)
    for tag, lam in (("rec", rec["x"]), ("recv", rec["vec"])):
        x, u, obj = recover(ga, lam)
        assert rel_err(x, rec[f"{tag}_x"]) < 1e-12
        assert rel_err(u, rec[f"{tag}_u"]) < 1e-12
        assert abs(obj - float(rec[f"{tag}_obj"])) <= 1e-11 * max(1.0, abs(float(rec[f"{tag}_obj"])))
        ref = rec[f"{tag}_kkt"]
        got = np.array(kkt(ga, lam, rec[f"{tag}_x"], rec[f"{tag}_u"]))
        scale = max(1.0, float(np.max(np.abs(rec[f"{tag}_x"]))), float(np.max(np.abs(lam))))
        assert np.all(np.abs(got - ref) <= 1e-12 * scale + 1e-9 * np.abs(ref)), (got, ref)


@pytest.mark.parametrize("name", GOLDEN_NAMES)
def test_oracle_recovery_matches_reference(name):
    _oracle_check(name)


@pytest.mark.gpu
@pytest.mark.parametrize("name", GOLDEN_NAMES)
def test_gpu_recovery_matches_reference(name):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2304_04980_b200 import GpuSchurOperator, kkt_residual, recover_solution

    ga, rec = load_golden(name)
    op = GpuSchurOperator(ga, rec["L"], rec["S"])
    for tag, lam in (("rec", rec["x"]), ("recv", rec["vec"])):
        sol = recover_solution(op, lam)
        assert rel_err(sol.x_flat, rec[f"{tag}_x"]) < 1e-12
        assert rel_err(sol.u_flat, rec[f"{tag}_u"]) < 1e-12
        ref_obj = float(rec[f"{tag}_obj"])
        assert abs(sol.objective_value - ref_obj) <= 1e-11 * max(1.0, abs(ref_obj))
        got = np.array(kkt_residual(op, sol))
        ref = rec[f"{tag}_kkt"]
        scale = max(1.0, float(np.max(np.abs(rec[f"{tag}_x"]))), float(np.max(np.abs(lam))))
        assert np.all(np.abs(got - ref) <= 1e-12 * scale + 1e-9 * np.abs(ref)), (got, ref)
        # state/input views
        lay = op.layout
        assert sol.state(0, 0).shape == (lay.T + 1, lay.n)
        assert sol.input(0, 0).shape == (lay.T, lay.m)


@pytest.mark.gpu
def test_gpu_recovery_headline_vs_oracle():
    """Full headline size: recovery and residuals of a random multiplier vector agree with
    the numpy restatement; on device tensors the outputs stay on the device."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle.gridlq_oracle import kkt, recover
    from paper_2304_04980_b200 import GpuSchurOperator, generators, kkt_residual, recover_solution

    ga = generators.config4(0)
    op = GpuSchurOperator(ga)
    lam = np.random.default_rng(3).standard_normal(op.dim)
    x, u, obj = recover(ga, lam)
    sol = recover_solution(op, torch.tensor(lam, device="cuda"))
    assert sol.x_flat.is_cuda and sol.u_flat.is_cuda
    assert rel_err(sol.x_flat.cpu().numpy(), x) < 1e-12
    assert rel_err(sol.u_flat.cpu().numpy(), u) < 1e-12
    assert abs(sol.objective_value - obj) <= 1e-10 * abs(obj)
    got = np.array(kkt_residual(op, sol))
    ref = np.array(kkt(ga, lam, sol.x_flat.cpu().numpy(), sol.u_flat.cpu().numpy()))
    assert np.all(np.abs(got - ref) <= 1e-12 * np.max(np.abs(x)) + 1e-9 * ref)
