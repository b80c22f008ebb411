"""Stage-slab sharded PCGM (paper_2304_04980_b200/slab.py).

CPU tier: the partition, the slab windows and the host-side PCG / halo / reduction logic,
with the oracle standing in for a slab's local compute (test-only), in one process and over
gloo with world_size 2.  GPU tier: the same solves with every slab on its own gq_ctx.
Parity rule as everywhere else: iterates 1e-9 relative, residual history
1e-9 + 1e-14 h0, equal step counts."""

import os
import socket

import numpy as np
import pytest
import torch

from conftest import load_golden, rel_err
from oracle.gridlq_oracle import Oracle
from paper_2304_04980_b200 import BreakdownError, MaxIterationsExceeded
from paper_2304_04980_b200.slab import SlabComm, SlabPcg, make_slabs, slab_arrays, slab_bounds
from test_oracle_golden import check_run

SMALL = ["boundary", "cg", "config1", "irrigation", "msd_ref", "odd_kn", "odd_kn_n4",
         "odd_n1", "sparse", "time_varying", "warm", "config5r", "config3r_l4"]


class OracleSlabOps:
    """Test-only stand-in for DeviceSlabOps: the CPU restatement on the slab's window."""

    def __init__(self, sub, inner_sweeps):
        self.o = Oracle(sub, inner_sweeps, 1)

    def delta(self, x):
        return torch.from_numpy(self.o.apply_delta(x.numpy()))

    def outer(self, x):
        return torch.from_numpy(self.o.apply_outer(x.numpy()))

    def inner(self, r):
        return torch.from_numpy(self.o.apply_precond(r.numpy()))


def _run(ga, rec, comm, factory=OracleSlabOps):
    solver = SlabPcg(ga, inner_sweeps=rec["L"], outer_sweeps=rec["S"], comm=comm,
                     ops_factory=factory, precondition=bool(rec["precond"]))
    try:
        x, rep = solver.solve(ga.offset, tol=rec["tol"], max_steps=rec["max_steps"],
                              x0=rec.get("x0"))
    except MaxIterationsExceeded as exc:
        x, rep = exc.iterate, exc.report
    return solver, x, rep


def test_slab_bounds():
    for T in (1, 2, 5, 20, 200):
        for p in range(1, min(T + 1, 9) + 1):
            b = slab_bounds(T, p)
            assert b[0][0] == 0 and b[-1][1] == T + 1
            assert all(b[i][1] == b[i + 1][0] for i in range(p - 1))
            sizes = [hi - lo for lo, hi in b]
            assert min(sizes) >= 1 and max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        slab_bounds(3, 5)
    with pytest.raises(ValueError):
        slab_bounds(3, 0)


def test_slab_windows_reproduce_global_rows():
    """Delta, Xi~ and the inner sweeps of a slab window equal the global operators on the
    owned rows once the halos hold the neighbours' stages (time-varying classes)."""
    ga, rec = load_golden("time_varying")
    full = Oracle(ga, 2, 1)
    rng = np.random.default_rng(3)
    v = rng.standard_normal(ga.dim)
    gd, go, gp = full.apply_delta(v), full.apply_outer(v), full.apply_precond(v)
    for p in (2, 3, ga.T + 1):
        for sl in make_slabs(ga, p):
            sub = slab_arrays(ga, sl)
            assert sub.T == sl.b - sl.a - 1
            o = Oracle(sub, 2, 1)
            loc = v[sl.a * sl.nh:sl.b * sl.nh]
            assert np.allclose(o.apply_delta(loc)[sl.own], gd[sl.global_own], rtol=0, atol=1e-13)
            assert np.allclose(o.apply_outer(loc)[sl.own], go[sl.global_own], rtol=0, atol=1e-13)
            # the inner sweeps are stage-local: no halo needed
            assert np.allclose(o.apply_precond(loc)[sl.own], gp[sl.global_own], rtol=0, atol=1e-13)


@pytest.mark.parametrize("name", SMALL)
@pytest.mark.parametrize("slabs", [2, 3])
def test_slab_pcg_in_process(name, slabs):
    ga, rec = load_golden(name)
    if slabs > ga.T + 1:
        pytest.skip("fewer stages than slabs")
    solver, x, rep = _run(ga, rec, SlabComm(slabs))
    check_run(name, rec, x, rep.residual_inf_history, rep.steps, rep.converged, {})
    from paper_2304_04980_b200 import COUNT_KEYS

    if name != "msd_ref_cg":
        got = np.array([rep.op_counts[k] for k in COUNT_KEYS])
        assert np.array_equal(got, rec["op_counts"])
    # one exchange per Delta apply and per extra outer sweep
    pcs = rep.steps + (1 if rec.get("x0") is not None else 0)
    n_prec = (1 + (rep.steps - 1 if rep.converged else rep.steps)) if rec["precond"] else 0
    assert solver.comm.exchanges == pcs + n_prec * (rec["S"] - 1)


def test_slab_every_stage_its_own_slab():
    ga, rec = load_golden("time_varying")
    _, x, rep = _run(ga, rec, SlabComm(ga.T + 1))
    check_run("time_varying", rec, x, rep.residual_inf_history, rep.steps, rep.converged, {})


def test_slab_errors():
    ga, rec = load_golden("config1")
    with pytest.raises(ValueError, match="even"):
        SlabPcg(ga, inner_sweeps=3, comm=SlabComm(2), ops_factory=OracleSlabOps)
    s = SlabPcg(ga, comm=SlabComm(2), ops_factory=OracleSlabOps)
    from paper_2304_04980_b200 import DimensionMismatchError

    with pytest.raises(DimensionMismatchError):
        s.solve(np.zeros(ga.dim + 1))
    bad = ga.offset.copy()
    bad[5] = np.nan
    with pytest.raises(ValueError):
        s.solve(bad)
    with pytest.raises(ValueError):
        s.solve(ga.offset, tol=0.0)
    with pytest.raises(ValueError):
        s.solve(ga.offset, max_steps=0)
    with pytest.raises(MaxIterationsExceeded) as ei:
        s.solve(ga.offset, tol=1e-30, max_steps=3)
    assert ei.value.iterations == 3 and ei.value.report.steps == 3
    # a negated operator has negative curvature: BreakdownError like pcg.py:103-107
    class Neg(OracleSlabOps):
        def delta(self, x):
            return -super().delta(x)

    neg = SlabPcg(ga, comm=SlabComm(2), ops_factory=Neg, precondition=False)
    with pytest.raises(BreakdownError):
        neg.solve(ga.offset)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, ws, port, name, slabs, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        ga, rec = load_golden(name)
        comm = SlabComm.from_env(slabs)
        solver, x, rep = _run(ga, rec, comm)
        out[rank] = (np.asarray(x).tolist(), list(rep.residual_inf_history), rep.steps,
                     rep.converged, solver.comm.local)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,slabs", [("config1", 2), ("time_varying", 4), ("warm", 2),
                                        ("config5r", 2)])
def test_slab_pcg_gloo(name, slabs):
    """world_size 2 over gloo: halos by isend/irecv, scalars by all_reduce; the result is
    the golden one and bitwise the in-process one (slab-order reductions)."""
    import torch.multiprocessing as mp

    ws = 2
    out = mp.Manager().list([None] * ws)
    mp.spawn(_gloo_worker, args=(ws, _free_port(), name, slabs, out), nprocs=ws, join=True)
    ga, rec = load_golden(name)
    x0, h0, s0, c0, l0 = out[0]
    x1, h1, s1, c1, l1 = out[1]
    assert sorted(l0 + l1) == list(range(slabs)) and not set(l0) & set(l1)
    assert x0 == x1 and h0 == h1 and s0 == s1 and c0 == c1
    check_run(name, rec, np.array(x0), h0, s0, c0, {})
    _, xi, repi = _run(ga, rec, SlabComm(slabs))
    assert np.array_equal(np.asarray(xi), np.array(x0))
    assert list(repi.residual_inf_history) == h0


# ---- GPU tier: the product path (each slab on its own gq_ctx) -------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("name", SMALL + ["config2", "config4r", "config3r"])
@pytest.mark.parametrize("slabs", [2, 3])
@pytest.mark.parametrize("native", [True, False])
def test_gpu_slab_pcg(name, slabs, native):
    """Both drivers (native stage-slab phases; composed applies) against the golden runs."""
    ga, rec = load_golden(name)
    if slabs > ga.T + 1:
        pytest.skip("fewer stages than slabs")
    solver = SlabPcg(ga, inner_sweeps=rec["L"], outer_sweeps=rec["S"],
                     comm=SlabComm(slabs, device=torch.device("cuda")),
                     precondition=bool(rec["precond"]), native=native)
    try:
        x, rep = solver.solve(ga.offset, tol=rec["tol"], max_steps=rec["max_steps"],
                              x0=rec.get("x0"))
    except MaxIterationsExceeded as exc:
        x, rep = exc.iterate, exc.report
    check_run(name, rec, x, rep.residual_inf_history, rep.steps, rep.converged, {})


@pytest.mark.gpu
def test_gpu_native_slab_callback_and_errors():
    """Native driver: per-step callback iterates match the golden snapshots; a budget
    exhausted run raises MaxIterationsExceeded with the iterate; every stage its own slab."""
    ga, rec = load_golden("config1")
    snaps = {}
    solver = SlabPcg(ga, comm=SlabComm(3, device=torch.device("cuda")))
    with pytest.raises(MaxIterationsExceeded) as ei:
        solver.solve(ga.offset, tol=rec["tol"], max_steps=rec["max_steps"],
                     callback=lambda k, x, r: snaps.__setitem__(k, x.copy()))
    check_run("config1", rec, ei.value.iterate, ei.value.report.residual_inf_history,
              ei.value.report.steps, ei.value.report.converged,
              {int(s): snaps[int(s)] for s in rec["snap_steps"] if int(s) in snaps})
    assert sorted(snaps) == list(range(1, rec["steps"] + 1))
    ga, rec = load_golden("time_varying")
    solver = SlabPcg(ga, comm=SlabComm(ga.T + 1, device=torch.device("cuda")))
    x, rep = solver.solve(ga.offset, tol=rec["tol"], max_steps=rec["max_steps"])
    check_run("time_varying", rec, x, rep.residual_inf_history, rep.steps, rep.converged, {})


@pytest.mark.gpu
def test_gpu_slabs_match_single_context():
    """A mid-size MSD grid (n = 2, the headline construction) split into 4 slabs against the
    one-context graph solve: same iterates to 1e-9, same history."""
    from paper_2304_04980_b200 import GpuNestedJacobiPreconditioner, GpuSchurOperator, pcg_solve
    from paper_2304_04980_b200.generators import msd_case

    ga = msd_case(48, 40, 30, seed=1)
    op = GpuSchurOperator(ga)
    pc = GpuNestedJacobiPreconditioner(op)
    try:
        x1, r1 = pcg_solve(op, pc, ga.offset, tol=1e-300, max_steps=25)
    except MaxIterationsExceeded as exc:
        x1, r1 = exc.iterate, exc.report
    for native, graph in ((True, True), (True, False), (False, None)):
        solver = SlabPcg(ga, comm=SlabComm(4, device=torch.device("cuda")), native=native,
                         graph=graph)
        try:
            x2, r2 = solver.solve(ga.offset, tol=1e-300, max_steps=25)
        except MaxIterationsExceeded as exc:
            x2, r2 = exc.iterate, exc.report
        assert r2.steps == r1.steps == 25
        assert rel_err(x2, x1) < 1e-9
        h1, h2 = np.array(r1.residual_inf_history), np.array(r2.residual_inf_history)
        assert np.all(np.abs(h2 - h1) <= 1e-9 * h1 + 1e-14 * h1[0])


# ---- native driver host logic (halo routing and scalar reductions) on CPU -----------------

class _FakeNative:
    """Stands in for _NativeSlab on CPU: a reference-order window vector per halo vector
    id; gq_slab_pack / gq_slab_unpack move one stage between it and a halo buffer."""

    def __init__(self, sl, value):
        self.sl = sl
        self.vec = {w: torch.zeros(sl.local_dim, dtype=torch.float64) for w in (0, 1, 2)}
        for w in self.vec:   # owned stages carry (global stage, vector id, value)
            for t in range(sl.lo, sl.hi):
                self.vec[w][sl.stage(t)] = 1000.0 * t + 10.0 * w + torch.arange(sl.nh) * 1e-3
        self.send = {k: torch.empty(sl.nh, dtype=torch.float64) for k in (0, 1)}
        self.recv = {k: torch.empty(sl.nh, dtype=torch.float64) for k in (0, 1)}
        self.scalar = {w: torch.tensor([value + w], dtype=torch.float64) for w in (0, 1, 2)}

    def _buf(self, ptr, others):
        for n in others:
            for b in list(n.send.values()) + list(n.recv.values()):
                if b.data_ptr() == ptr.value:
                    return b
        raise KeyError(ptr)

    def call(self, fn, which, t, ptr):
        lt = self.sl.a + t
        if fn == "gq_slab_pack":
            self._buf(ptr, [self]).copy_(self.vec[which][self.sl.stage(lt)])
        else:
            self.vec[which][self.sl.stage(lt)] = self._buf(ptr, _FakeNative.everyone)


def _native_logic(comm, ga):
    s = object.__new__(SlabPcg)
    s.comm, s.slabs = comm, make_slabs(ga, comm.n)
    _FakeNative.everyone = []
    s.nat = {k: _FakeNative(s.slabs[k], float(k + 1)) for k in comm.local}
    _FakeNative.everyone = list(s.nat.values())
    for w in (0, 1, 2):
        s._nexchange(w)
    s._nreduce(0, "sum")        # curvature
    s._nreduce_res_mu()         # max|r| and q.r in one collective
    out = {}
    for k, nat in s.nat.items():
        sl = nat.sl
        halos = {}
        for t in (sl.lo - 1, sl.hi):
            if sl.a <= t < sl.b:
                halos[t] = [nat.vec[w][sl.stage(t)].tolist() for w in (0, 1, 2)]
        out[k] = (halos, float(nat.scalar[0]), float(nat.scalar[1]), float(nat.scalar[2]))
    return out


def _check_native_logic(out, ga, n):
    nh = ga.K * ga.N * ga.n
    for k, (halos, ssum, smax, smu) in out.items():
        assert ssum == sum(float(j + 1) for j in range(n))          # curvature slot: summed
        assert smax == float(n) + 1.0                                # residual slot: max
        assert smu == sum(float(j + 3) for j in range(n))           # q.r slot: summed
        for t, vs in halos.items():
            for w, v in enumerate(vs):
                assert np.allclose(v, 1000.0 * t + 10.0 * w + np.arange(nh) * 1e-3)


def test_native_exchange_and_reduce_in_process():
    ga, _ = load_golden("config1")
    out = _native_logic(SlabComm(4), ga)
    assert sorted(out) == [0, 1, 2, 3]
    _check_native_logic(out, ga, 4)


def _native_gloo_worker(rank, ws, port, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        ga, _ = load_golden("config1")
        res = _native_logic(SlabComm.from_env(4), ga)
        out[rank] = {k: v for k, v in res.items()}
    finally:
        dist.destroy_process_group()


def test_native_exchange_and_reduce_gloo():
    """The native driver's halo routing (pack -> isend/irecv -> unpack across processes,
    device copy inside one) and scalar reductions, world_size 2 with 2 slabs each."""
    import torch.multiprocessing as mp

    out = mp.Manager().list([None, None])
    mp.spawn(_native_gloo_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    ga, _ = load_golden("config1")
    merged = {}
    for part in out:
        merged.update(part)
    assert sorted(merged) == [0, 1, 2, 3]
    _check_native_logic(merged, ga, 4)


@pytest.mark.gpu
def test_gpu_native_slabs_headline_size():
    """BASELINE config 4 at full size (256 x 256, T = 200) in 4 native slabs against the
    one-context graph solve over 6 steps: iterates to 1e-9, history to 1e-9."""
    from paper_2304_04980_b200 import GpuNestedJacobiPreconditioner, GpuSchurOperator, pcg_solve
    from paper_2304_04980_b200.generators import config4

    ga = config4(0)
    rhs = torch.from_numpy(ga.offset).cuda()
    op = GpuSchurOperator(ga)
    pc = GpuNestedJacobiPreconditioner(op)
    with pytest.raises(MaxIterationsExceeded) as e1:
        pcg_solve(op, pc, rhs, tol=1e-300, max_steps=6)
    x1 = e1.value.iterate.cpu().numpy()
    h1 = np.array(e1.value.report.residual_inf_history)
    del op, pc
    solver = SlabPcg(ga, comm=SlabComm(4, device=torch.device("cuda")))
    with pytest.raises(MaxIterationsExceeded) as e2:
        solver.solve(rhs, tol=1e-300, max_steps=6)
    # the captured step graph is reused by the next solve on the same solver
    with pytest.raises(MaxIterationsExceeded) as e3:
        solver.solve(rhs, tol=1e-300, max_steps=6)
    assert torch.equal(e3.value.iterate, e2.value.iterate)
    x2 = e2.value.iterate.cpu().numpy()
    h2 = np.array(e2.value.report.residual_inf_history)
    assert rel_err(x2, x1) < 1e-9
    assert np.all(np.abs(h2 - h1) <= 1e-9 * h1 + 1e-14 * h1[0])


def _gpu_gloo_worker(rank, ws, port, name, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        ga, rec = load_golden(name)
        solver = SlabPcg(ga, inner_sweeps=rec["L"], outer_sweeps=rec["S"],
                         comm=SlabComm.from_env(2 * ws, device=torch.device("cuda")),
                         precondition=bool(rec["precond"]))
        assert solver.native and not solver.graph
        try:
            x, rep = solver.solve(ga.offset, tol=rec["tol"], max_steps=rec["max_steps"],
                                  x0=rec.get("x0"))
        except MaxIterationsExceeded as exc:
            x, rep = exc.iterate, exc.report
        out[rank] = (np.asarray(x).tolist(), list(rep.residual_inf_history), rep.steps,
                     rep.converged)
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["config1", "time_varying", "warm", "config5r", "cg"])
def test_gpu_native_slabs_two_processes(name):
    """The native driver across processes: 2 processes x 2 slabs on the one GPU, halos and
    scalars through gloo (host-staged; the kernels never wait on each other, only the host
    does).  Same golden parity as everywhere; both processes return the same solve."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    out = ctx.Manager().list([None, None])
    mp.start_processes(_gpu_gloo_worker, args=(2, _free_port(), name, out), nprocs=2,
                       join=True, start_method="spawn")
    ga, rec = load_golden(name)
    x0, h0, s0, c0 = out[0]
    x1, h1, s1, c1 = out[1]
    assert x0 == x1 and h0 == h1 and s0 == s1 and c0 == c1
    check_run(name, rec, np.array(x0), h0, s0, c0, {})
