"""Generate golden parity fixtures by running the REFERENCE itself -- test infrastructure.

Imports ``gridlq`` read-only from /root/reference/pkg/src (this container only; the GPU
box never sees /root/reference), builds each case, and records into
``tests/golden/<case>.npz``:

* the problem as GridArrays fields (what the B200 path and the oracle consume);
* the reference's omega~ (``build_stacked(...).offset``) and flop counters
  (``SchurOperator.matvec_flops``/``outer_coupling_flops``,
  ``PairSplitting.inner_coupling_flops``, ``NestedJacobiPreconditioner.pair_solve_flops``
  / ``apply_flops``);
* Delta v, Xi~ v, Omega~ v, Phi~^-1 v and the preconditioner apply on a seeded v;
* a ``pcg_solve`` run: residual history, final iterate, iterates at selected steps
  (through ``callback``), step count, convergence flag, op_counts.

Run:  python oracle/make_golden.py   (writes tests/golden/, takes ~2-3 minutes)
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import gridlq  # noqa: E402

import cases  # noqa: E402
from paper_2304_04980_b200 import generators as G  # noqa: E402
from paper_2304_04980_b200.problem import arrays_from_problem, arrays_to_problem  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
COUNT_KEYS = gridlq.pcg.COUNT_KEYS


def run_case(name, problem, L=2, S=2, tol=None, rel_tol=None, max_steps=None, precond=True,
             x0_seed=None, snap=(1,), vec_seed=0):
    t0 = time.time()
    ga = arrays_from_problem(problem)
    stacked = gridlq.build_stacked(problem)
    schur = gridlq.build_schur(stacked)
    pc = gridlq.NestedJacobiPreconditioner(schur, L, S)
    rhs = stacked.offset
    if rel_tol is not None:
        tol = rel_tol * float(np.max(np.abs(rhs)))
    rng = np.random.default_rng(vec_seed)
    v = rng.standard_normal(schur.dim)
    rec = dict(
        K=ga.K, N=ga.N, T=ga.T, n=ga.n, m=ga.m, A=ga.A, B=ga.B, R=ga.R, C=ga.C,
        cmask=ga.cmask, Q=ga.Q, dyn_class=ga.dyn_class, cost_class=ga.cost_class,
        offset=ga.offset, ref_offset=rhs, L=L, S=S, tol=tol,
        max_steps=-1 if max_steps is None else max_steps, precond=int(precond),
        matvec_flops=schur.matvec_flops, outer_coupling_flops=schur.outer_coupling_flops,
        inner_coupling_flops=pc.splitting.inner_coupling_flops,
        pair_solve_flops=pc.pair_solve_flops, apply_flops=pc.apply_flops,
        vec=v, delta=schur.apply(v), outer=schur.apply_outer_coupling(v),
        inner=pc.splitting.apply_inner_coupling(v), pair=pc._pair_solves(v),
    )
    if L % 2 == 0:
        rec["prec"] = pc.apply(v)
    x0 = None
    if x0_seed is not None:
        x0 = 0.1 * np.random.default_rng(x0_seed).standard_normal(schur.dim)
        rec["x0"] = x0
    snaps = {}

    def cb(step, x, r):
        if step in snap:
            snaps[step] = (x.copy(), r.copy())

    status = "ok"
    try:
        x, rep = gridlq.pcg_solve(schur, pc if precond else None, rhs, tol=tol,
                                  max_steps=max_steps, x0=x0, callback=cb)
    except gridlq.MaxIterationsExceeded as exc:
        x, rep, status = exc.iterate, exc.report, "max_steps"
    rec.update(
        x=x, hist=np.array(rep.residual_inf_history), steps=rep.steps,
        converged=int(rep.converged), status=status,
        op_counts=np.array([rep.op_counts[k] for k in COUNT_KEYS]),
        snap_steps=np.array(sorted(snaps), dtype=np.int64),
        snap_x=np.array([snaps[s][0] for s in sorted(snaps)]),
        snap_r=np.array([snaps[s][1] for s in sorted(snaps)]),
    )
    # primal recovery + KKT residuals (recovery.py:50-80) at the solve's final multipliers
    # and at the random vector (non-trivial dynamics residual)
    for tag, lam in (("rec", x), ("recv", v)):
        sol = gridlq.recover_solution(stacked, lam)
        rec[f"{tag}_x"] = sol.x_flat
        rec[f"{tag}_u"] = sol.u_flat
        rec[f"{tag}_obj"] = sol.objective_value
        rec[f"{tag}_kkt"] = np.array(gridlq.kkt_residual(stacked, sol))
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **rec)
    print(f"{name}: dim={schur.dim} steps={rep.steps} conv={rep.converged} "
          f"({time.time() - t0:.1f}s)", flush=True)


def run_nbjm(name, problem, L=2, tol=1e-9, max_outer=50000):
    """Standalone nested Jacobi solve (nested_jacobi.py:124-151) -> tests/golden/nbjm_<name>.npz."""
    t0 = time.time()
    ga = arrays_from_problem(problem)
    stacked = gridlq.build_stacked(problem)
    schur = gridlq.build_schur(stacked)
    pc = gridlq.NestedJacobiPreconditioner(schur, L, 1)
    rhs = stacked.offset
    try:
        x, outers = gridlq.nbjm_solve(pc, rhs, tol=tol, max_outer=max_outer)
        converged = 1
    except gridlq.MaxIterationsExceeded as exc:
        x, outers, converged = exc.iterate, exc.iterations, 0
    rec = dict(
        K=ga.K, N=ga.N, T=ga.T, n=ga.n, m=ga.m, A=ga.A, B=ga.B, R=ga.R, C=ga.C,
        cmask=ga.cmask, Q=ga.Q, dyn_class=ga.dyn_class, cost_class=ga.cost_class,
        offset=ga.offset, ref_offset=rhs, L=L, tol=tol, max_outer=max_outer, x=x,
        outers=outers, converged=converged)
    np.savez_compressed(os.path.join(OUT, f"nbjm_{name}.npz"), **rec)
    print(f"nbjm_{name}: dim={schur.dim} L={L} outers={outers} conv={converged} "
          f"({time.time() - t0:.1f}s)", flush=True)


def main():
    os.makedirs(OUT, exist_ok=True)
    only = set(sys.argv[1:])

    def want(n):
        return not only or n in only

    if want("nbjm"):
        msd = gridlq.generate_msd_case
        run_nbjm("msd_l2", msd(3, 3, 3, seed=1), L=2, tol=1e-9)
        run_nbjm("msd_l4", msd(3, 3, 3, seed=1), L=4, tol=1e-9)
        run_nbjm("msd_budget", msd(3, 3, 3, seed=1), L=2, tol=1e-9, max_outer=3)
        run_nbjm("msd5_l2", msd(5, 5, 5, seed=0), L=2, tol=1e-9)
        run_nbjm("msd_odd_l2", msd(5, 3, 4, seed=2), L=2, tol=1e-9)
        run_nbjm("irr_l1", gridlq.generate_irrigation_case(2, 2, 2), L=1, tol=1e-10)
        run_nbjm("irr_l3", gridlq.generate_irrigation_case(3, 4, 3, seed=2), L=3, tol=1e-9)
        return
    if want("config1"):
        run_case("config1", arrays_to_problem(G.config1(0)), tol=1e-30, max_steps=50,
                 snap=(1, 25, 50))
    if want("config2"):
        run_case("config2", arrays_to_problem(G.config2(0)), rel_tol=1e-10, snap=(1, 10, 40))
    if want("config3r"):
        run_case("config3r", arrays_to_problem(G.config3(0, K=8, N=8, T=20)), L=2, S=3,
                 tol=1e-30, max_steps=200, snap=(1, 20, 100, 200))
    if want("config3r_l4"):
        run_case("config3r_l4", arrays_to_problem(G.config3(1, K=6, N=6, T=10)), L=4, S=3,
                 rel_tol=1e-10, snap=(1, 5))
    if want("config4r"):
        run_case("config4r", arrays_to_problem(G.config4(0, K=24, N=24, T=20)), tol=1e-30,
                 max_steps=40, snap=(1, 20, 40))
    if want("config5r"):
        run_case("config5r", arrays_to_problem(G.config5(0, K=6, N=12, T=5)), rel_tol=1e-10,
                 snap=(1, 10))
    if want("config5r_s4l4"):
        run_case("config5r_s4l4", arrays_to_problem(G.config5(2, K=4, N=6, T=4)), L=4, S=4,
                 rel_tol=1e-10, snap=(1,))
    if want("odd_kn"):
        run_case("odd_kn", arrays_to_problem(G.random_case(5, 3, 4, 2, 1, seed=3)), tol=1e-30,
                 max_steps=30, snap=(1, 30))
    if want("odd_kn_n4"):
        run_case("odd_kn_n4", arrays_to_problem(
            G.random_case(3, 5, 3, 4, 2, seed=4, q_diag_range=(1, 10))), rel_tol=1e-10)
    if want("odd_n1"):
        run_case("odd_n1", arrays_to_problem(G.random_case(7, 1, 6, 1, 1, seed=8)),
                 rel_tol=1e-10)
    if want("boundary"):
        run_case("boundary", cases.boundary_problem(), tol=1e-9, snap=(1, 2))
        # problem files written by the reference itself (JSON ingestion parity)
        gridlq.save_problem(cases.boundary_problem(), os.path.join(OUT, "boundary_problem.json"))
    if want("time_varying"):
        run_case("time_varying", cases.time_varying(), rel_tol=1e-10, snap=(1, 3))
        gridlq.save_problem(cases.time_varying(), os.path.join(OUT, "time_varying_problem.json"))
    if want("sparse"):
        run_case("sparse", cases.sparse_couplings(), rel_tol=1e-10, snap=(1,))
    if want("uncoupled"):
        run_case("uncoupled", cases.uncoupled(), tol=1e-9, precond=False)
    if want("scalar"):
        run_case("scalar", cases.scalar_chain(), tol=1e-12)
    if want("msd_ref"):
        run_case("msd_ref", gridlq.generate_msd_case(3, 3, 3, seed=1), tol=1e-9, snap=(1, 5))
    if want("msd_ref_cg"):
        run_case("msd_ref_cg", gridlq.generate_msd_case(3, 3, 3, seed=1), tol=1e-9,
                 precond=False, snap=(1, 10))
    if want("irrigation"):
        run_case("irrigation", gridlq.generate_irrigation_case(3, 4, 3, seed=2), tol=1e-9)
    if want("warm"):
        run_case("warm", arrays_to_problem(G.config1(1)), tol=1e-30, max_steps=12,
                 x0_seed=5, snap=(1, 12))
    if want("cg"):
        run_case("cg", arrays_to_problem(G.config1(2)), tol=1e-30, max_steps=30,
                 precond=False, snap=(1, 30))


if __name__ == "__main__":
    main()
