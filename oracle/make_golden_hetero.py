"""Golden fixture for mixed subsystem dimensions, produced by running the REFERENCE itself on
tests/cases.hetero_problem (test infrastructure; this container only):
tests/golden/hetero/hetero.npz holds the reference's omega~, flop counters, Delta v and the
preconditioner apply on a seeded v, a pcg_solve run (iterate, history, steps, op_counts) and
the recovered trajectory with its objective and KKT residuals.

Run:  python oracle/make_golden_hetero.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import gridlq  # noqa: E402

import cases  # noqa: E402


def main():
    p = cases.hetero_problem()
    assert gridlq.validate(p) == []
    st = gridlq.build_stacked(p)
    sc = gridlq.build_schur(st)
    pc = gridlq.NestedJacobiPreconditioner(sc, 2, 2)
    v = np.random.default_rng(0).standard_normal(sc.dim)
    tol = 1e-10 * float(np.max(np.abs(st.offset)))
    x, rep = gridlq.pcg_solve(sc, pc, st.offset, tol=tol)
    sol = gridlq.recover_solution(st, x)
    res = gridlq.kkt_residual(st, sol)
    rec = dict(
        dim=sc.dim, ref_offset=st.offset, v=v, delta_v=sc.apply(v), precond_v=pc.apply(v),
        outer_v=sc.apply_outer_coupling(v), matvec_flops=sc.matvec_flops,
        outer_coupling_flops=sc.outer_coupling_flops, pair_solve_flops=pc.pair_solve_flops,
        apply_flops=pc.apply_flops, tol=tol, x=x, hist=np.array(rep.residual_inf_history),
        steps=rep.steps, converged=int(rep.converged),
        op_keys=np.array(list(rep.op_counts)), op_vals=np.array([rep.op_counts[k] for k in rep.op_counts]),
        sol_x=sol.x_flat, sol_u=sol.u_flat, objective=sol.objective_value, kkt=np.array(res))
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "hetero", "hetero.npz"), **rec)
    print("hetero: dim", sc.dim, "steps", rep.steps, "objective", sol.objective_value, "kkt", res)


if __name__ == "__main__":
    main()
