"""Host mirror of the reference's PCGM interface, executed by libgridlq_b200.so.

Drop-in for the reference's hot path (``gridlq/pcg.py``, ``gridlq/nested_jacobi.py``,
``gridlq/kkt_assembly.py``):

* ``GpuSchurOperator``  -- duck type of ``SchurOperator`` (``.dim``, ``.matvec_flops``,
  ``.outer_coupling_flops``, ``.apply(x, pool=None)``, ``.apply_outer_coupling(x)``)
* ``GpuNestedJacobiPreconditioner`` -- duck type of ``NestedJacobiPreconditioner``
  (constructor ``(schur, inner_sweeps=2, outer_sweeps=2)``, ``.apply(r, pool=None)``,
  ``.apply_flops``, ``.pair_solve_flops``, ``.inner_sweep``-level pieces)
* ``pcg_solve`` / ``cg_solve`` / ``SolveReport`` / ``COUNT_KEYS`` -- same signatures,
  return values, exceptions and op_counts bookkeeping as ``pcg.py:19-156``.

Because both duck types are honoured, the reference's own ``gridlq.pcg_solve`` can also
drive the GPU operators (one device apply per call); the fast path is this module's
``pcg_solve``, which runs the whole loop on the device.
"""

from __future__ import annotations

import atexit
import ctypes
import os
import threading
import time
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .counts import counters
from .errors import BreakdownError, DimensionMismatchError, MaxIterationsExceeded
from .problem import GridArrays, as_arrays, rhs_offset_device

COUNT_KEYS = (
    "operator_apply",
    "curvature_dot",
    "solution_update",
    "residual_update",
    "residual_norm",
    "preconditioner_apply",
    "precondition_dot",
    "direction_update",
)


@dataclass
class SolveReport:
    """Mirror of ``pcg.py:31-47``."""

    steps: int
    residual_inf_history: list
    converged: bool
    tolerance: float
    wall_time_s: float
    op_counts: dict = field(default_factory=dict)

    @property
    def final_residual(self):
        return self.residual_inf_history[-1] if self.residual_inf_history else float("nan")

    @property
    def flops_per_step(self):
        total = sum(self.op_counts.values())
        return total / self.steps if self.steps else 0.0


def _torch_cuda(x):
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor) and x.is_cuda


class _Vec:
    """A vector argument at the C-ABI: host numpy (float64, contiguous) or a CUDA torch
    tensor (float64, contiguous) passed by device pointer."""

    def __init__(self, x, dim, name):
        if _torch_cuda(x):
            if x.dtype != __import__("torch").float64 or x.dim() != 1 or x.numel() != dim:
                raise DimensionMismatchError(f"{name} must be a float64 vector of length {dim}")
            self.obj = x.contiguous()
            self.ptr = self.obj.data_ptr()
            self.device = True
        else:
            arr = np.ascontiguousarray(np.asarray(x, dtype=float))
            if arr.ndim != 1 or arr.shape[0] != dim:
                raise DimensionMismatchError(
                    f"{name} has shape {arr.shape}, operator dimension is {dim}")
            self.obj = arr
            self.ptr = arr.ctypes.data
            self.device = False

    def like(self):
        if self.device:
            import torch
            return torch.empty_like(self.obj)
        return np.empty_like(self.obj)


class _PinnedPool:
    """Page-locked host buffers for result arrays.  A result array is a numpy view of a ctypes
    array over ``gq_host_alloc`` memory; when the last reference to it (or to any view of it)
    goes, the buffer comes back here instead of being unlocked -- page-locking 211 MB costs more
    than a 100-step solve, re-using a locked buffer costs nothing.  At most ``keep`` free buffers
    per size are held; the rest are released.  Page-locked memory is a scarce resource: once
    ``max(limit, 4 buffers)`` bytes are locked (results the caller still holds plus the pool),
    further results go to ordinary pageable arrays."""

    def __init__(self, keep=2, limit=2 << 30):
        self.keep = keep
        self.limit = limit
        self.locked = 0
        self.free = {}
        self.closed = False
        atexit.register(self.close)

    def _release(self, nbytes, ptr):
        self.locked -= nbytes
        try:
            _lib.load().gq_host_free(ctypes.c_void_p(ptr))
        except Exception:      # interpreter shutdown
            pass

    def _give(self, nbytes, ptr):
        lst = self.free.setdefault(nbytes, [])
        if self.closed or len(lst) >= self.keep:
            self._release(nbytes, ptr)
        else:
            lst.append(ptr)

    def take(self, n):
        """A float64 array of n entries in page-locked memory, or None."""
        if self.closed or os.environ.get("GQ_NO_PINNED_RESULT") == "1":
            return None
        nbytes = 8 * int(n)
        lst = self.free.get(nbytes)
        if lst:
            ptr = lst.pop()
        else:
            if self.locked + nbytes > max(self.limit, 4 * nbytes):
                return None
            ptr = _lib.load().gq_host_alloc(nbytes)
            if not ptr:
                return None
            self.locked += nbytes
        buf = (ctypes.c_double * int(n)).from_address(ptr)
        weakref.finalize(buf, self._give, nbytes, ptr)
        return np.frombuffer(buf, dtype=np.float64)

    def close(self):
        self.closed = True
        for nbytes, lst in self.free.items():
            while lst:
                self._release(nbytes, lst.pop())


_pinned = _PinnedPool()


def _touch_pages(arr):
    """Write one byte per 4 KiB page (from several threads, ``gq_touch_pages``) so a fresh
    host array is resident before the device-to-host copy lands in it."""
    _lib.load().gq_touch_pages(ctypes.c_void_p(arr.ctypes.data), arr.nbytes)


def _ptr(out):
    return out.data_ptr() if _torch_cuda(out) else out.ctypes.data


class _Context:
    """Owns one gq_ctx (device setup of a problem)."""

    def __init__(self, ga: GridArrays, inner_sweeps=2, outer_sweeps=2):
        lib = _lib.load()
        self.ga = ga
        self._keep = []

        def dptr(a):
            a = np.ascontiguousarray(a, dtype=np.float64)
            self._keep.append(a)
            return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))

        def iptr(a):
            a = np.ascontiguousarray(a, dtype=np.int32)
            self._keep.append(a)
            return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))

        desc = _lib.GqProblemDesc(
            K=ga.K, N=ga.N, T=ga.T, n=ga.n, m=ga.m, n_dyn=len(ga.A), n_cost=len(ga.Q),
            dyn_class=iptr(ga.dyn_class), cost_class=iptr(ga.cost_class),
            A=dptr(ga.A), B=dptr(ga.B), R=dptr(ga.R), C=dptr(ga.C), Q=dptr(ga.Q))
        handle = ctypes.c_void_p()
        _lib.check(lib.gq_create(ctypes.byref(desc), int(inner_sweeps), int(outer_sweeps),
                                 ctypes.byref(handle)), "setup")
        self._keep.clear()
        self.lib = lib
        self.h = handle
        self.dim = int(lib.gq_dim(handle))
        self.L, self.S = int(inner_sweeps), int(outer_sweeps)
        self.embed = None   # embed.Embedding when the problem has mixed dimensions

    def set_sweeps(self, inner, outer):
        if (inner, outer) != (self.L, self.S):
            _lib.check(self.lib.gq_set_sweeps(self.h, int(inner), int(outer)))
            self.L, self.S = int(inner), int(outer)

    def unary(self, fn, x, name="x"):
        if self.embed is not None:
            x = self.embed.expand_x(x, name)
        v = _Vec(x, self.dim, name)
        out = v.like()
        _lib.check(getattr(self.lib, fn)(self.h, v.ptr, _ptr(out)), fn)
        return out if self.embed is None else self.embed.restrict_x(out)

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            try:
                self.lib.gq_destroy(h)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass
            self.h = None


class GpuSchurOperator:
    """The reduced multiplier operator Delta on the device (``kkt_assembly.py:326-484``).

    ``problem`` is a GridLQProblem (reference data model) or GridArrays.  The right-hand
    side omega~ of ``build_stacked`` (``kkt_assembly.py:275-301``) is ``.offset``.
    """

    def __init__(self, problem, inner_sweeps=2, outer_sweeps=2):
        self._embed = None
        if not isinstance(problem, GridArrays):
            from .embed import Embedding, needs_embedding
            from .problem import problem_messages
            if needs_embedding(problem):
                # mixed state/input dimensions (grid_problem.py:103-141), or a uniform state
                # dimension without compiled kernels (5, 6, 7): solve the padded uniform
                # problem, map vectors at the interface (embed.py)
                msgs = problem_messages(problem)
                if msgs:
                    raise ValueError("invalid problem: " + "; ".join(msgs))
                self._embed = Embedding(problem)
                self._hetero_problem = problem
                problem = self._embed.padded_problem(problem)
        self.arrays = as_arrays(problem)
        self._problem = None if isinstance(problem, GridArrays) else problem
        self._ctx = _Context(self.arrays, inner_sweeps, outer_sweeps)
        self._ctx.embed = self._embed
        self.dim = self._ctx.dim if self._embed is None else self._embed.dim
        self.layout = self.arrays.layout if self._embed is None else self._embed.layout()
        self.pairs = self.layout.pairs
        self.offset = (self.arrays.offset if self._embed is None
                       else self._embed.restrict_x(self.arrays.offset))
        self._counts = {}

    def offset_device(self):
        """omega~ as a CUDA tensor: built by the ``gq_build_offset`` kernel when the operator
        was made from a GridLQProblem (``kkt_assembly.py:275-301``), uploaded otherwise."""
        import torch

        if self._problem is not None:
            off = rhs_offset_device(self._problem, self.arrays.n)
            return off if self._embed is None else self._embed.restrict_x(off)
        return torch.as_tensor(self.arrays.offset, device="cuda")

    def counts(self, inner_sweeps=2, outer_sweeps=2):
        key = (inner_sweeps, outer_sweeps)
        if key not in self._counts:
            emb = self._embed
            self._counts[key] = counters(self.arrays, inner_sweeps, outer_sweeps,
                                         nd=None if emb is None else emb.nd)
        return self._counts[key]

    @property
    def matvec_flops(self):
        return self.counts()["matvec_flops"]

    @property
    def outer_coupling_flops(self):
        return self.counts()["outer_coupling_flops"]

    def apply(self, x, pool=None):
        """Delta x (``kkt_assembly.py:389-403``); ``pool`` is accepted and ignored."""
        return self._ctx.unary("gq_apply_delta", x)

    def apply_outer_coupling(self, x):
        """Xi~ x (``kkt_assembly.py:414-425``)."""
        return self._ctx.unary("gq_apply_outer_coupling", x)


def apply_delta(schur: GpuSchurOperator, x, pool=None):
    return schur.apply(x, pool=pool)


def build_schur(problem, inner_sweeps=2, outer_sweeps=2) -> GpuSchurOperator:
    return GpuSchurOperator(problem, inner_sweeps, outer_sweeps)


class GpuNestedJacobiPreconditioner:
    """Fixed-budget nested block Jacobi map (``nested_jacobi.py:23-161``) on the device.

    The pair-chain block Cholesky factors are built once, on the device, when the
    operator's context is created; they do not depend on the budgets.
    """

    def __init__(self, schur: GpuSchurOperator, inner_sweeps=2, outer_sweeps=2, splitting=None):
        if inner_sweeps < 1 or outer_sweeps < 1:
            raise ValueError("sweep budgets must be at least 1")  # nested_jacobi.py:33-34
        if not isinstance(schur, GpuSchurOperator):
            raise TypeError("GpuNestedJacobiPreconditioner needs a GpuSchurOperator")
        self.schur = schur
        self.inner_sweeps = int(inner_sweeps)
        self.outer_sweeps = int(outer_sweeps)

    @property
    def dim(self):
        return self.schur.dim

    def _counts(self):
        return self.schur.counts(self.inner_sweeps, self.outer_sweeps)

    @property
    def pair_solve_flops(self):
        return self._counts()["pair_solve_flops"]

    @property
    def apply_flops(self):
        return self._counts()["apply_flops"]

    def _select(self):
        self.schur._ctx.set_sweeps(self.inner_sweeps, self.outer_sweeps)

    def apply(self, r, pool=None):
        """nested_jacobi.py:105-122: S outer x L inner sweeps from zero."""
        if self.inner_sweeps % 2:
            raise ValueError(
                "preconditioner use requires an even inner budget "
                f"(got {self.inner_sweeps}); odd budgets are standalone-only")
        self._select()
        if isinstance(r, np.ndarray) and r.ndim == 2:
            return np.stack([self.apply(r[:, c]) for c in range(r.shape[1])], axis=1)
        return self.schur._ctx.unary("gq_apply_precond", r, "r")

    def solve(self, rhs, tol=1e-9, max_outer=50000, pool=None):
        """Standalone nested Jacobi iteration (``nested_jacobi.py:124-151``) on the device.

        Outer sweeps run until the successive-iterate infinity norm drops below ``tol``;
        inner sweeps are warm-started from the current outer iterate, so any inner budget
        >= 1 is allowed.  Returns ``(solution, outer sweep count)``; raises
        MaxIterationsExceeded carrying the last iterate when the budget runs out.  ``pool``
        is accepted and ignored.
        """
        ctx = self.schur._ctx
        max_outer = int(max_outer)
        msg = f"nested Jacobi did not converge within {max_outer} outer sweeps"
        emb = ctx.embed
        if emb is not None:
            rhs = emb.expand_x(rhs, "rhs")
        v = _Vec(rhs, ctx.dim, "rhs")
        if max_outer < 1:            # the reference loop never runs
            raise MaxIterationsExceeded(msg, iterate=None, iterations=max_outer)
        self._select()
        out = v.like()
        outers = ctypes.c_int64()
        rc = ctx.lib.gq_nbjm_solve(ctx.h, v.ptr, float(tol), max_outer, _ptr(out),
                                   ctypes.byref(outers))
        if emb is not None:
            out = emb.restrict_x(out)
        if rc == _lib.GQ_MAX_ITER:
            raise MaxIterationsExceeded(msg, iterate=out, iterations=max_outer)
        _lib.check(rc, "nbjm_solve")
        return out, int(outers.value)

    def pair_solves(self, rhs):
        """Phi~^-1 rhs over every (pair, stage) chain (nested_jacobi.py:65-77)."""
        return self.schur._ctx.unary("gq_pair_solve", rhs, "rhs")

    def apply_inner_coupling(self, x):
        """Omega~ x (kkt_assembly.py:645-662)."""
        return self.schur._ctx.unary("gq_apply_inner_coupling", x)


def nbjm_solve(precond: GpuNestedJacobiPreconditioner, rhs, tol=1e-9, max_outer=50000,
               pool=None):
    """Standalone nested-Jacobi solve with an existing preconditioner's factors and budgets
    (``nested_jacobi.py:155-159``)."""
    return precond.solve(rhs, tol=tol, max_outer=max_outer, pool=pool)


def _op_counts(dim, matvec, precond_flops, steps, converged, warm):
    """pcg.py:76-131 bookkeeping in closed form (test_pcg.py:141-152 semantics)."""
    c = dict.fromkeys(COUNT_KEYS, 0.0)
    loop_precond = steps - 1 if converged else steps
    c["operator_apply"] = float(matvec * (steps + (1 if warm else 0)))
    c["curvature_dot"] = float(dim * steps)
    c["solution_update"] = float(dim * steps)
    c["residual_update"] = float(dim * steps)
    c["residual_norm"] = float(dim * steps)
    c["preconditioner_apply"] = float(precond_flops * (1 + loop_precond))
    c["precondition_dot"] = float(dim * (1 + loop_precond))
    c["direction_update"] = float(dim * loop_precond)
    return c


def pcg_solve(schur, preconditioner, rhs, tol=1e-9, max_steps=None, x0=None, pool=None,
              callback=None):
    """Preconditioned conjugate gradient (``pcg.py:50-149``) run on the B200.

    Same contract as the reference: returns ``(x, SolveReport)``; raises
    DimensionMismatchError / ValueError on bad input, BreakdownError on non-positive
    curvature and MaxIterationsExceeded (with ``iterate``, ``iterations``, ``report``)
    when the budget runs out.  ``callback(step, x, r)`` is honoured by stepping the
    device loop one step at a time (slow; parity/debug use).
    """
    if not isinstance(schur, GpuSchurOperator):
        raise TypeError("pcg_solve here runs GpuSchurOperator on the device; use the "
                        "reference gridlq.pcg_solve for host operators")
    if preconditioner is not None and (not isinstance(preconditioner, GpuNestedJacobiPreconditioner)
                                       or preconditioner.schur is not schur):
        raise TypeError("preconditioner must be a GpuNestedJacobiPreconditioner on `schur`")
    ctx = schur._ctx
    dim = schur.dim
    # shape checks here; the non-finite check (pcg.py:65-66) runs on the device inside
    # gq_pcg_start and surfaces as ValueError through _lib.check
    is_dev = _torch_cuda(rhs)
    if is_dev:
        if rhs.dim() != 1 or rhs.numel() != dim:
            raise DimensionMismatchError("right-hand side does not match operator dimension")
    else:
        rhs = np.asarray(rhs, dtype=float)
        if rhs.ndim != 1 or rhs.shape[0] != dim:
            raise DimensionMismatchError("right-hand side does not match operator dimension")
    if tol <= 0:
        raise ValueError("tolerance must be positive")
    if max_steps is None:
        max_steps = dim + 50
    if max_steps < 1:
        raise ValueError("need at least one step")
    use_pc = preconditioner is not None
    if use_pc:
        if preconditioner.inner_sweeps % 2:
            raise ValueError(
                "preconditioner use requires an even inner budget "
                f"(got {preconditioner.inner_sweeps}); odd budgets are standalone-only")
        preconditioner._select()
    start = time.perf_counter()
    emb = ctx.embed
    if emb is not None:      # mixed dimensions: the device works on the padded vectors
        rhs = emb.expand_x(rhs, "rhs")
        x0 = emb.expand_x(x0, "x0") if x0 is not None else None
    rv = _Vec(rhs, ctx.dim, "rhs")
    x0v = _Vec(x0, ctx.dim, "x0") if x0 is not None else None
    lib = ctx.lib
    _lib.check(lib.gq_pcg_start(ctx.h, rv.ptr, x0v.ptr if x0v else None, int(use_pc)), "pcg")
    steps = ctypes.c_int64()
    conv = ctypes.c_int32()
    # large host results land in page-locked memory (from a pool); failing that, in a fresh
    # array whose pages are faulted in while the device iterates (ctypes drops the GIL)
    x = None
    if not rv.device and 8 * ctx.dim >= (8 << 20):
        x = _pinned.take(ctx.dim)
    pinned = x is not None
    if x is None:
        x = rv.like()
    if callback is None:
        toucher = None
        if not rv.device and not pinned and x.nbytes >= (8 << 20):
            toucher = threading.Thread(target=_touch_pages, args=(x,), daemon=True)
            toucher.start()
        status = lib.gq_pcg_run(ctx.h, float(tol), int(max_steps), ctypes.byref(steps),
                                ctypes.byref(conv))
        if toucher is not None:
            toucher.join()
    else:
        status = _lib.GQ_OK
        for k in range(1, int(max_steps) + 1):
            status = lib.gq_pcg_run(ctx.h, float(tol), k, ctypes.byref(steps), ctypes.byref(conv))
            if status == _lib.GQ_BREAKDOWN or steps.value < k:
                break
            xk, rk = rv.like(), rv.like()
            _lib.check(lib.gq_pcg_read(ctx.h, _lib.GQ_VEC_X, _ptr(xk)))
            _lib.check(lib.gq_pcg_read(ctx.h, _lib.GQ_VEC_R, _ptr(rk)))
            if emb is not None:
                xk, rk = emb.restrict_x(xk), emb.restrict_x(rk)
            callback(steps.value, xk, rk)
            if conv.value:
                break
    if status not in (_lib.GQ_OK, _lib.GQ_MAX_ITER, _lib.GQ_BREAKDOWN):
        _lib.check(status, "pcg")
    if status == _lib.GQ_BREAKDOWN:
        raise BreakdownError(_lib.last_error())
    nsteps = int(steps.value)
    _lib.check(lib.gq_pcg_read(ctx.h, _lib.GQ_VEC_X, _ptr(x)))
    if emb is not None:
        x = emb.restrict_x(x)
    hist = np.empty(nsteps)
    if nsteps:
        _lib.check(lib.gq_pcg_history(ctx.h, hist.ctypes.data, nsteps))
    converged = bool(conv.value)
    counts = _op_counts(dim, schur.matvec_flops,
                        preconditioner.apply_flops if use_pc else 0.0, nsteps, converged,
                        x0 is not None)
    report = SolveReport(steps=nsteps, residual_inf_history=[float(h) for h in hist],
                         converged=converged, tolerance=tol,
                         wall_time_s=time.perf_counter() - start, op_counts=counts)
    if not converged:
        raise MaxIterationsExceeded(
            f"conjugate gradient did not reach {tol:g} within {nsteps} steps "
            f"(residual {report.final_residual:.3e})",
            iterate=x, iterations=nsteps, report=report)
    return x, report


def cg_solve(schur, rhs, tol=1e-9, max_steps=None, x0=None, pool=None, callback=None):
    """Unpreconditioned conjugate gradient baseline (``pcg.py:152-156``)."""
    return pcg_solve(schur, None, rhs, tol=tol, max_steps=max_steps, x0=x0, pool=pool,
                     callback=callback)
