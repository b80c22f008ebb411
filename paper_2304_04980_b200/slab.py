"""Stage-slab sharded PCGM.

The reference solves the whole multiplier system in one process (``pcg.py:50-149``).  The
path partitions naturally along the stage axis t:

* Delta couples stage t only to t-1 and t+1 (``kkt_assembly.py:389-403``);
* the pair-chain solves and Omega~ are stage-local (``nested_jacobi.py:65-103``);
* Xi~ couples t to t +- 1 again (``kkt_assembly.py:414-425``);
* PCG itself needs three scalar reductions per step (``pcg.py:100,112,128``).

So each slab owns a contiguous stage range [lo, hi) and keeps one halo stage on each side
that has a neighbour.  A slab is an ordinary problem of its own: the stage window
[lo - 1, hi + 1) of the global data, with the global stage-class maps sliced to it.  Every
row that the slab owns then sees exactly the global operator blocks (its Psi_t, Xi_{t-1},
Xi_t and the pair factors of its class); only the halo rows differ, and those are never
read.  Per PCG step the slabs exchange one stage of the direction d (before Delta d) and
one stage of delta per extra outer sweep (before Xi~ delta): ``S`` halo exchanges of
``K*N*n`` doubles per side, plus the three scalar reductions.

Slabs map onto processes in contiguous blocks (one process per GPU, ``torch.distributed``
over NCCL for the halos and scalars; gloo on CPU for the host-logic tests).  Several slabs
may live in one process: their halos are device copies.  The composed driver sums per-slab
partials in slab order, so its runs are bitwise independent of the slab-to-process layout;
the native one reduces in-process first, then over the group.

Two drivers share this partition:

* native (the default on a GPU): every slab's ``gq_ctx`` runs the PCG step kernels of the
  one-GPU path in stage-slab mode (``gq_slab_*`` in include/gridlq_b200.h).  A step is six
  phases enqueued on the device stream; between them the halos move by pack -> NCCL
  send/recv (or a device copy) -> unpack and the partial scalars are reduced on the device
  (curvature and q.r summed, max|r| maxed).  The host never waits inside a step; it polls
  the convergence flag after 2, 4, ..., 64 steps like ``gq_pcg_run``.
* composed (``native=False``, or an ``ops_factory``): the step is written here with torch
  vector ops over three per-slab applies through the C ABI (``gq_apply_delta``,
  ``gq_apply_outer_coupling``, ``gq_apply_precond`` with one outer sweep).  It is the
  readable statement of the algorithm and the form the CPU tests drive, with the oracle
  standing in for the applies (test-only).
"""

from __future__ import annotations

import ctypes
import dataclasses
import time

import numpy as np

from .counts import counters
from .errors import BreakdownError, DimensionMismatchError, MaxIterationsExceeded
from .problem import GridArrays, as_arrays
from .solver import SolveReport, _op_counts


def slab_bounds(T: int, slabs: int) -> list:
    """Owned stage ranges [lo, hi) of ``slabs`` contiguous slabs over stages 0..T
    (sizes differ by at most one, the larger ones first)."""
    stages = T + 1
    if slabs < 1 or slabs > stages:
        raise ValueError(f"need 1 <= slabs <= T + 1 = {stages}, got {slabs}")
    base, extra = divmod(stages, slabs)
    out, lo = [], 0
    for s in range(slabs):
        hi = lo + base + (1 if s < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


@dataclasses.dataclass(frozen=True)
class Slab:
    """One slab: owned global stages [lo, hi), local window [a, b) = owned + halos."""

    index: int
    lo: int
    hi: int
    a: int
    b: int
    nh: int            # doubles per stage (K * N * n)

    @property
    def local_dim(self):
        return (self.b - self.a) * self.nh

    @property
    def own(self):
        """Owned part of a local vector (reference order: stages are contiguous)."""
        return slice((self.lo - self.a) * self.nh, (self.hi - self.a) * self.nh)

    @property
    def global_own(self):
        return slice(self.lo * self.nh, self.hi * self.nh)

    def stage(self, t):
        """Local slice of global stage t (t in [a, b))."""
        o = (t - self.a) * self.nh
        return slice(o, o + self.nh)


def make_slabs(ga: GridArrays, slabs: int) -> list:
    nh = ga.K * ga.N * ga.n
    out = []
    for s, (lo, hi) in enumerate(slab_bounds(ga.T, slabs)):
        out.append(Slab(s, lo, hi, max(lo - 1, 0), min(hi + 1, ga.T + 1), nh))
    return out


def slab_arrays(ga: GridArrays, sl: Slab) -> GridArrays:
    """The slab's window [a, b) as a problem of its own: same blocks, the global stage-class
    maps sliced to the window (``dyn_class`` covers the transitions a..b-2)."""
    return dataclasses.replace(
        ga, T=sl.b - sl.a - 1,
        dyn_class=np.ascontiguousarray(ga.dyn_class[sl.a:sl.b - 1]),
        cost_class=np.ascontiguousarray(ga.cost_class[sl.a:sl.b]),
        offset=np.ascontiguousarray(ga.offset[sl.a * sl.nh:sl.b * sl.nh]))


class DeviceSlabOps:
    """Local compute of one slab on the B200: its own gq_ctx, one outer sweep per
    preconditioner call (the outer loop runs in ``SlabPcg`` with halo exchanges)."""

    def __init__(self, sub: GridArrays, inner_sweeps: int):
        import torch

        from . import _lib
        from .solver import _Context

        self.ctx = _Context(sub, inner_sweeps, 1)
        # order the library's work after torch's on the same stream
        stream = torch.cuda.current_stream()
        _lib.check(self.ctx.lib.gq_set_stream(self.ctx.h, ctypes.c_void_p(stream.cuda_stream)))
        self.device = torch.device("cuda", torch.cuda.current_device())

    def delta(self, x):
        return self.ctx.unary("gq_apply_delta", x)

    def outer(self, x):
        return self.ctx.unary("gq_apply_outer_coupling", x)

    def inner(self, r):
        return self.ctx.unary("gq_apply_precond", r)


class _WarmStartOps:
    """Delta through a native slab's context (warm start only: r = rhs - Delta x0)."""

    def __init__(self, nat):
        self.nat = nat

    def delta(self, x):
        return self.nat.ctx.unary("gq_apply_delta", x)


class SlabComm:
    """Halo exchange and scalar reductions between the slabs of one partition.

    ``owner[s]`` is the process rank holding slab s; this process holds the slabs with
    ``owner[s] == rank``.  ``group`` is a torch.distributed process group (None: the
    default group when initialised, else a single process)."""

    def __init__(self, n_slabs: int, world: int = 1, rank: int = 0, group=None, device=None):
        import torch

        if n_slabs % world:
            raise ValueError(f"{n_slabs} slabs do not divide over {world} processes")
        per = n_slabs // world
        self.owner = [s // per for s in range(n_slabs)]
        self.rank, self.world, self.group = rank, world, group
        self.local = [s for s in range(n_slabs) if self.owner[s] == rank]
        self.n = n_slabs
        self.device = device if device is not None else torch.device("cpu")
        self.exchanges = 0
        # gloo carries host tensors only: the native driver stages its device halos and
        # scalars through the host (the multi-process GPU test; NCCL takes device buffers)
        self.host_staged = False
        if world > 1:
            import torch.distributed as dist

            self.host_staged = dist.get_backend(group) == "gloo"

    @classmethod
    def from_env(cls, n_slabs: int, group=None, device=None):
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized():
            return cls(n_slabs, dist.get_world_size(group), dist.get_rank(group), group, device)
        return cls(n_slabs, 1, 0, None, device)

    def exchange(self, slabs, vecs):
        """Fill every halo stage of ``vecs`` (slab -> local vector) from the neighbour's
        owned boundary stage.  Reads touch owned stages only and writes halo stages only,
        so the in-process copies need no ordering."""
        import torch
        import torch.distributed as dist

        self.exchanges += 1
        reqs, staged = [], []
        for s in self.local:
            sl = slabs[s]
            for nb, mine, theirs in ((s - 1, sl.lo - 1, sl.lo), (s + 1, sl.hi, sl.hi - 1)):
                if nb < 0 or nb >= self.n:
                    continue
                halo = vecs[s][sl.stage(mine)]            # my halo = their boundary stage
                if self.owner[nb] == self.rank:
                    halo.copy_(vecs[nb][slabs[nb].stage(mine)])
                else:
                    peer = self.owner[nb]
                    snd, rcv = vecs[s][sl.stage(theirs)], halo
                    if self.host_staged and halo.device.type != "cpu":
                        snd, rcv = snd.cpu(), torch.empty_like(halo, device="cpu")
                        staged.append((halo, rcv))
                    reqs.append(dist.P2POp(dist.isend, snd, peer, group=self.group))
                    reqs.append(dist.P2POp(dist.irecv, rcv, peer, group=self.group))
        # one NCCL group for all sends and receives: both directions in flight together
        for r in (dist.batch_isend_irecv(reqs) if reqs else []):
            r.wait()
        for halo, rcv in staged:
            halo.copy_(rcv)

    def _reduce(self, partials, op):
        import torch
        import torch.distributed as dist

        if self.world == 1:
            vals = [partials[s] for s in range(self.n)]
        else:
            buf = torch.zeros(self.n, dtype=torch.float64, device=self.device)
            for s in self.local:
                buf[s] = partials[s]
            dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=self.group)   # x + 0 is exact
            vals = buf.tolist()
        if op == "sum":
            acc = 0.0
            for v in vals:        # slab order: independent of the process layout
                acc += v
            return acc
        return max(vals)

    def sum(self, partials):
        return self._reduce(partials, "sum")

    def max(self, partials):
        return self._reduce(partials, "max")

    def gather(self, slabs, vecs, dim):
        """The global vector (every process gets it): owned parts summed into zeros."""
        import torch
        import torch.distributed as dist

        any_vec = vecs[self.local[0]]
        out = torch.zeros(dim, dtype=any_vec.dtype, device=any_vec.device)
        for s in self.local:
            out[slabs[s].global_own] = vecs[s][slabs[s].own]
        if self.world > 1:
            dist.all_reduce(out, op=dist.ReduceOp.SUM, group=self.group)
        return out


class _DevScalar:
    """A device double inside a gq_ctx, exposed to torch (``__cuda_array_interface__``)."""

    def __init__(self, ptr):
        self.__cuda_array_interface__ = {"shape": (1,), "typestr": "<f8", "data": (ptr, False),
                                         "version": 3}


class _NativeSlab:
    """One slab's gq_ctx in stage-slab mode, with its halo buffers and scalar views."""

    def __init__(self, sub: GridArrays, sl: Slab, inner_sweeps, outer_sweeps):
        import torch

        from . import _lib
        from .solver import _Context

        self.sl = sl
        self.ctx = _Context(sub, inner_sweeps, outer_sweeps)
        lib, h = self.ctx.lib, self.ctx.h
        stream = torch.cuda.current_stream()
        _lib.check(lib.gq_set_stream(h, ctypes.c_void_p(stream.cuda_stream)))
        _lib.check(lib.gq_slab_enable(h, sl.lo - sl.a, sl.hi - sl.a), "slab")
        self.scalar = {}
        for w in (_lib.GQ_SLAB_CURV, _lib.GQ_SLAB_RES, _lib.GQ_SLAB_MU):
            ptr = lib.gq_slab_scalar_ptr(h, w)
            self.scalar[w] = torch.as_tensor(_DevScalar(ptr), device="cuda")
        dev = torch.device("cuda", torch.cuda.current_device())
        self.send = {side: torch.empty(sl.nh, dtype=torch.float64, device=dev) for side in (0, 1)}
        self.recv = {side: torch.empty(sl.nh, dtype=torch.float64, device=dev) for side in (0, 1)}

    def call(self, fn, *args):
        from . import _lib

        _lib.check(getattr(self.ctx.lib, fn)(self.ctx.h, *args), fn)


class SlabPcg:
    """PCGM over a stage-slab partition (``pcg.py:50-149`` control flow).

    * ``native`` (default when no ``ops_factory`` is given): every slab's gq_ctx runs the
      step kernels in stage-slab mode; ``graph`` (default: all slabs in this process)
      replays the whole sharded step as one captured CUDA graph.
    * composed (``native=False``): torch vector ops over per-slab applies;
      ``ops_factory(sub_arrays, inner_sweeps)`` builds them (default ``DeviceSlabOps``; the
      tests pass an oracle-backed factory).
    * ``time_from`` (attribute, native only): when set to W, the next solve records CUDA
      events around its steps W..max_steps-1 into ``last_timed = (steps, ms)`` (bench.py).
    """

    def __init__(self, problem, slabs=None, inner_sweeps=2, outer_sweeps=2, comm=None,
                 ops_factory=None, precondition=True, native=None, graph=None):
        import torch

        self.arrays = as_arrays(problem)
        ga = self.arrays
        if precondition and inner_sweeps % 2:
            raise ValueError("preconditioner use requires an even inner budget "
                             f"(got {inner_sweeps}); odd budgets are standalone-only")
        if inner_sweeps < 1 or outer_sweeps < 1:
            raise ValueError("sweep budgets must be at least 1")
        if comm is None:
            dev = torch.device("cuda", torch.cuda.current_device()) if ops_factory is None \
                else torch.device("cpu")
            if slabs is None:
                import torch.distributed as dist

                slabs = dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1
            comm = SlabComm.from_env(slabs, device=dev)
        self.comm = comm
        self.slabs = make_slabs(ga, comm.n)
        self.L, self.S = int(inner_sweeps), int(outer_sweeps)
        self.precondition = precondition
        self.native = (ops_factory is None) if native is None else bool(native)
        if self.native and ops_factory is not None:
            raise ValueError("the native slab driver runs the device kernels; drop ops_factory")
        if self.native:
            # all native work runs on one dedicated stream (it is also the capture stream)
            self.stream = torch.cuda.Stream()
            with torch.cuda.stream(self.stream):
                self.nat = {s: _NativeSlab(slab_arrays(ga, self.slabs[s]), self.slabs[s], self.L,
                                           self.S) for s in comm.local}
            # one CUDA graph per sharded step when every slab is in this process
            self.graph = (comm.world == 1) if graph is None else bool(graph)
            self._graphs = {}
            # the composed applies are only needed for a warm start's r = rhs - Delta x0
            self.ops = {s: _WarmStartOps(self.nat[s]) for s in comm.local}
        else:
            factory = ops_factory or DeviceSlabOps
            self.ops = {s: factory(slab_arrays(ga, self.slabs[s]), self.L) for s in comm.local}
        self.dim = ga.dim
        self.device = comm.device if ops_factory is not None else \
            torch.device("cuda", torch.cuda.current_device())

    # -- local vectors ------------------------------------------------------------------
    def _scatter(self, v):
        """Global vector -> {slab: local vector}, owned stages filled, halos zero."""
        import torch

        out = {}
        for s in self.comm.local:
            sl = self.slabs[s]
            loc = torch.zeros(sl.local_dim, dtype=torch.float64, device=self.device)
            loc[sl.own] = v[sl.global_own]
            out[s] = loc
        return out

    def _dot(self, a, b):
        return self.comm.sum({s: float(a[s][self.slabs[s].own] @ b[s][self.slabs[s].own])
                              for s in self.comm.local})

    def precond(self, r):
        """q = P r (``nested_jacobi.py:105-122``): delta^0 = inner(r); for the further outer
        sweeps delta = inner(r + Xi~ delta) with the delta halos exchanged first."""
        delta = {s: self.ops[s].inner(r[s]) for s in self.comm.local}
        for _ in range(self.S - 1):
            self.comm.exchange(self.slabs, delta)
            delta = {s: self.ops[s].inner(r[s] + self.ops[s].outer(delta[s]))
                     for s in self.comm.local}
        return delta

    def delta(self, x):
        self.comm.exchange(self.slabs, x)
        return {s: self.ops[s].delta(x[s]) for s in self.comm.local}

    # -- the solve ----------------------------------------------------------------------
    def solve(self, rhs, tol=1e-9, max_steps=None, x0=None, callback=None):
        """Same contract as ``pcg_solve`` (``pcg.py:50-149``): returns (x, SolveReport);
        DimensionMismatchError / ValueError on bad input, BreakdownError on non-positive
        curvature, MaxIterationsExceeded carrying the iterate and report."""
        import torch

        dim = self.dim
        host = not (isinstance(rhs, torch.Tensor) and rhs.device.type != "cpu")
        rv = torch.as_tensor(np.asarray(rhs, dtype=float) if host and not isinstance(rhs, torch.Tensor)
                             else rhs, dtype=torch.float64)
        if rv.dim() != 1 or rv.numel() != dim:
            raise DimensionMismatchError("right-hand side does not match operator dimension")
        if tol <= 0:
            raise ValueError("tolerance must be positive")
        if max_steps is None:
            max_steps = dim + 50
        if max_steps < 1:
            raise ValueError("need at least one step")
        start = time.perf_counter()
        rv = rv.to(self.device)
        if not bool(torch.isfinite(rv).all()):     # pcg.py:65-66, checked where rv lives now
            raise ValueError("right-hand side contains non-finite entries")
        if self.native:
            cur = torch.cuda.current_stream()
            self.stream.wait_stream(cur)
            try:
                with torch.cuda.stream(self.stream):
                    return self._solve_body(rv, x0, tol, max_steps, host, start, callback)
            finally:      # results (and the iterate of MaxIterationsExceeded) are on that stream
                cur.wait_stream(self.stream)
        return self._solve_body(rv, x0, tol, max_steps, host, start, callback)

    def _solve_body(self, rv, x0, tol, max_steps, host, start, callback):
        import torch

        dim = self.dim
        own = {s: self.slabs[s].own for s in self.comm.local}
        loc = self.comm.local
        r = self._scatter(rv)
        x0s = None
        if x0 is None:
            x = {s: torch.zeros_like(r[s]) for s in loc}
        else:
            x0v = torch.as_tensor(np.asarray(x0, dtype=float) if not isinstance(x0, torch.Tensor)
                                  else x0, dtype=torch.float64).to(self.device)
            if x0v.dim() != 1 or x0v.numel() != dim:
                raise DimensionMismatchError("x0 does not match operator dimension")
            x = self._scatter(x0v)
            ax = self.delta(x)
            for s in loc:
                r[s][own[s]] = r[s][own[s]] - ax[s][own[s]]
            x0s = x
        if self.native:
            return self._solve_native(r, x0s, tol, int(max_steps), host, start, callback)
        d = self.precond(r) if self.precondition else {s: r[s].clone() for s in loc}
        mu = self._dot(d, r)
        hist, steps, converged = [], 0, False
        for _ in range(int(max_steps)):
            y = self.delta(d)
            curv = self._dot(y, d)
            if curv <= 0.0:
                raise BreakdownError(f"non-positive curvature {curv:.3e} at step {steps + 1}")
            alpha = mu / curv
            for s in loc:
                o = own[s]
                x[s][o] += alpha * d[s][o]
                r[s][o] = r[s][o] - alpha * y[s][o]
            res = self.comm.max({s: float(r[s][own[s]].abs().max()) for s in loc})
            hist.append(res)
            steps += 1
            if callback is not None:
                callback(steps, self._out(x, host), self._out(r, host))
            if res < tol:
                converged = True
                break
            q = self.precond(r) if self.precondition else r
            mu_next = self._dot(q, r)
            beta = mu_next / mu
            d = {s: q[s] + beta * d[s] for s in loc}
            mu = mu_next
        return self._finish(self._out(x, host), hist, steps, converged, tol, start,
                            x0 is not None)

    # -- native stage-slab mode ------------------------------------------------------------
    def _nexchange(self, which):
        """Halo exchange of a device work vector (gq_slab_pack / NCCL or copy / unpack)."""
        import torch
        import torch.distributed as dist

        comm, nat, slabs = self.comm, self.nat, self.slabs
        comm.exchanges += 1
        sides = {}
        for s in comm.local:
            sl = slabs[s]
            for side, nb, mine, theirs in ((0, s - 1, sl.lo - 1, sl.lo), (1, s + 1, sl.hi, sl.hi - 1)):
                if 0 <= nb < comm.n:
                    sides.setdefault(s, []).append((side, nb, mine - sl.a, theirs - sl.a))
                    nat[s].call("gq_slab_pack", which, theirs - sl.a,
                                ctypes.c_void_p(nat[s].send[side].data_ptr()))
        reqs, later = [], []
        for s, lst in sides.items():
            for side, nb, halo_t, _ in lst:
                if comm.owner[nb] == comm.rank:
                    src = nat[nb].send[1 - side]
                    nat[s].call("gq_slab_unpack", which, halo_t, ctypes.c_void_p(src.data_ptr()))
                else:
                    peer = comm.owner[nb]
                    snd, rcv = nat[s].send[side], nat[s].recv[side]
                    if comm.host_staged:     # gloo moves host tensors only
                        snd, rcv = snd.cpu(), torch.empty_like(rcv, device="cpu")
                    reqs.append(dist.P2POp(dist.isend, snd, peer, group=comm.group))
                    reqs.append(dist.P2POp(dist.irecv, rcv, peer, group=comm.group))
                    later.append((s, side, halo_t, rcv))
        for q in (dist.batch_isend_irecv(reqs) if reqs else []):
            q.wait()
        for s, side, halo_t, rcv in later:
            if rcv.device.type == "cpu":
                nat[s].recv[side].copy_(rcv)
            nat[s].call("gq_slab_unpack", which, halo_t, ctypes.c_void_p(nat[s].recv[side].data_ptr()))

    def _gather_combine(self, part, ops):
        """Combine a vector of per-process partials over the process group: all-gathered and
        folded in rank order on the device (ops[i] in {"sum", "max"} per entry), so every
        collective of the slab step follows one deterministic rule whatever the slab-to-
        process mapping (NCCL's own all-reduce order is not fixed)."""
        import torch
        import torch.distributed as dist

        if self.comm.world == 1:
            return part
        buf = part.cpu() if self.comm.host_staged else part
        k = buf.numel()
        allp = torch.empty(self.comm.world * k, dtype=torch.float64, device=buf.device)
        dist.all_gather_into_tensor(allp, buf, group=self.comm.group)
        allp = allp.view(self.comm.world, k).to(part.device)
        tot = [allp[0, i] for i in range(k)]
        for w in range(1, self.comm.world):
            tot = [torch.maximum(tot[i], allp[w, i]) if ops[i] == "max" else tot[i] + allp[w, i]
                   for i in range(k)]
        return torch.stack(tot)

    def _nreduce(self, which, op):
        """Combine one device scalar over all slabs: local slabs in slab order, then the
        processes in rank order (_gather_combine)."""
        import torch

        vals = [self.nat[s].scalar[which] for s in self.comm.local]
        if len(vals) == 1 and self.comm.world == 1:
            return
        # a torch-allocated scalar carries the collective (the slots live in library memory)
        tot = vals[0].clone()
        for v in vals[1:]:
            tot = tot + v if op == "sum" else torch.maximum(tot, v)
        tot = self._gather_combine(tot, (op,))
        for v in vals:
            v.copy_(tot)

    def _nreduce_res_mu(self):
        """max|r| (max) and q.r (sum) in ONE collective: every process contributes its
        (max, sum) pair, all-gathered and combined in rank order on the device."""
        import torch

        from . import _lib

        res = [self.nat[s].scalar[_lib.GQ_SLAB_RES] for s in self.comm.local]
        mu = [self.nat[s].scalar[_lib.GQ_SLAB_MU] for s in self.comm.local]
        if len(res) == 1 and self.comm.world == 1:
            return
        pair = torch.cat([res[0], mu[0]])
        for r_, m_ in zip(res[1:], mu[1:]):
            pair = torch.stack([torch.maximum(pair[0], r_[0]), pair[1] + m_[0]])
        pair = self._gather_combine(pair, ("max", "sum"))
        for r_, m_ in zip(res, mu):
            r_.copy_(pair[0:1])
            m_.copy_(pair[1:2])

    def _nphase(self, kind, s=0):
        for k in self.comm.local:
            self.nat[k].call("gq_slab_phase", kind, s)

    def _comm(self, fn, *args):
        """Run one exchange / reduction; with ``comm_events`` set (a list, eager steps only)
        bracket it with CUDA events on the solver stream so bench.py can report the step's
        communication time per rank."""
        ce = getattr(self, "comm_events", None)
        if ce is None:
            return fn(*args)
        import torch

        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn(*args)
        e1.record()
        ce.append((e0, e1))

    def _nstep(self, S):
        from . import _lib

        self._comm(self._nexchange, _lib.GQ_SLAB_VEC_D)
        self._nphase(_lib.GQ_SLAB_DELTA)
        self._comm(self._nreduce, _lib.GQ_SLAB_CURV, "sum")
        self._nphase(_lib.GQ_SLAB_UPDATE)
        for s in range(S):
            self._nphase(_lib.GQ_SLAB_OUTER, s)
            if s < S - 1:
                self._comm(self._nexchange, _lib.GQ_SLAB_VEC_DL0 + s % 2)
        self._comm(self._nreduce_res_mu)
        self._nphase(_lib.GQ_SLAB_DIRECTION)

    def _solve_native(self, r, x0s, tol, max_steps, host, start, callback=None):
        import torch

        from . import _lib

        loc = self.comm.local
        S = self.S if self.precondition else 1
        for s in loc:
            xp = ctypes.c_void_p(x0s[s].data_ptr()) if x0s is not None else None
            self.nat[s].call("gq_slab_start", ctypes.c_void_p(r[s].data_ptr()), xp,
                             int(self.precondition), float(tol), int(max_steps))
        for s in range(S):
            self._nphase(_lib.GQ_SLAB_INIT_OUTER, s)
            if s < S - 1:
                self._nexchange(_lib.GQ_SLAB_VEC_DL0 + s % 2)
        self._nreduce(_lib.GQ_SLAB_MU, "sum")
        self._nphase(_lib.GQ_SLAB_INIT_FINISH)
        first = self.nat[loc[0]]
        # a host result: fault its pages in while the device iterates (as pcg_solve does)
        xhost, toucher = None, None
        if host and self.comm.world == 1 and callback is None:
            import threading

            from .solver import _touch_pages

            xhost = np.empty(self.dim)
            toucher = threading.Thread(target=_touch_pages, args=(xhost,), daemon=True)
            toucher.start()
        step, done = ctypes.c_int64(), ctypes.c_int32()
        conv, brk = ctypes.c_int32(), ctypes.c_int32()
        issued, chunk = 0, 1 if callback is not None else 2
        use_graph = self.graph and callback is None
        # device timing of the steps after the first `time_from` (bench.py): CUDA events on
        # the solver stream around exactly those steps
        tf = getattr(self, "time_from", None)
        ev = None
        while True:
            todo = min(chunk, max_steps - issued)
            for _ in range(todo):
                if tf is not None and issued + _ == tf:
                    ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                    ev[0].record()
                g = self._graphs.get(S) if use_graph else None
                if g is not None:
                    g.replay()
                else:
                    self._nstep(S)      # eager (also warms the launch caches before capture)
                    if use_graph:
                        g = torch.cuda.CUDAGraph()
                        with torch.cuda.graph(g, stream=self.stream,
                                              capture_error_mode="thread_local"):
                            self._nstep(S)
                        self._graphs[S] = g
            issued += todo
            if ev is not None and issued >= max_steps:
                ev[1].record()
            first.call("gq_slab_status", ctypes.byref(step), ctypes.byref(done),
                       ctypes.byref(conv), ctypes.byref(brk))
            if callback is not None and not brk.value and step.value == issued:
                callback(int(step.value), self._nread(_lib.GQ_VEC_X, host),
                         self._nread(_lib.GQ_VEC_R, host))
            if done.value or step.value >= max_steps or issued >= max_steps:
                break
            if callback is None:
                chunk = min(chunk * 2, 64)
        if ev is not None and issued >= max_steps:
            ev[1].synchronize()
            self.last_timed = (max_steps - tf, ev[0].elapsed_time(ev[1]))
        steps = int(step.value)
        hist = np.empty(steps)
        if steps:
            first.call("gq_pcg_history", hist.ctypes.data, steps)
        if brk.value:
            raise BreakdownError(f"non-positive curvature at step {steps + 1}; operator or "
                                 "preconditioner is not positive definite")
        if toucher is not None:
            toucher.join()
        xg = self._nread(_lib.GQ_VEC_X, host, out=xhost)
        converged = bool(conv.value)
        return self._finish(xg, hist.tolist(), steps, converged, tol, start, x0s is not None)

    def _nread(self, which, host, out=None):
        """Global x or r assembled from the slabs' owned stages."""
        import torch

        if host and self.comm.world == 1:
            # host result in one process: the library's staged export per slab (a direct
            # device -> pageable copy of a 211 MB vector costs ~95 ms here)
            if out is None:
                out = np.empty(self.dim)
            for s in self.comm.local:
                sl = self.slabs[s]
                if sl.local_dim == self.dim:
                    self.nat[s].call("gq_pcg_read", which, ctypes.c_void_p(out.ctypes.data))
                else:
                    tmp = np.empty(sl.local_dim)
                    self.nat[s].call("gq_pcg_read", which, ctypes.c_void_p(tmp.ctypes.data))
                    out[sl.global_own] = tmp[sl.own]
            return out
        vs = {}
        for s in self.comm.local:
            vs[s] = torch.empty(self.slabs[s].local_dim, dtype=torch.float64, device=self.device)
            self.nat[s].call("gq_pcg_read", which, ctypes.c_void_p(vs[s].data_ptr()))
        return self._out(vs, host)

    def _finish(self, xg, hist, steps, converged, tol, start, warm):
        ga = self.arrays
        cnt = counters(ga, self.L, self.S)
        counts = _op_counts(self.dim, cnt["matvec_flops"],
                            cnt["apply_flops"] if self.precondition else 0.0, steps, converged,
                            warm)
        report = SolveReport(steps=steps, residual_inf_history=[float(h) for h in hist],
                             converged=converged, tolerance=tol,
                             wall_time_s=time.perf_counter() - start, op_counts=counts)
        if not converged:
            raise MaxIterationsExceeded(
                f"conjugate gradient did not reach {tol:g} within {steps} steps "
                f"(residual {report.final_residual:.3e})",
                iterate=xg, iterations=steps, report=report)
        return xg, report

    def _out(self, v, host):
        g = self.comm.gather(self.slabs, v, self.dim)
        return g.cpu().numpy() if host else g


def pcg_solve_slabs(problem, rhs, tol=1e-9, max_steps=None, x0=None, inner_sweeps=2,
                    outer_sweeps=2, slabs=None, precondition=True, callback=None, native=None):
    """Stage-slab sharded ``pcg_solve``: ``slabs`` slabs over the processes of the default
    torch.distributed group (one process per GPU), or all in this process when no group is
    initialised.  Returns the global iterate on every process."""
    solver = SlabPcg(problem, slabs=slabs, inner_sweeps=inner_sweeps, outer_sweeps=outer_sweeps,
                     precondition=precondition, native=native)
    return solver.solve(rhs, tol=tol, max_steps=max_steps, x0=x0, callback=callback)
