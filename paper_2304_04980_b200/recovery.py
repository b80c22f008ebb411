"""Primal recovery and first-order optimality residuals on the device
(reference ``gridlq/recovery.py:24-80``).

``recover_solution(schur, multipliers)`` evaluates x = -Q^-1 (A~' lam), u = -R^-1 (B~' lam)
and the objective 0.5 (x'Qx + u'Ru); ``kkt_residual(schur, sol)`` the infinity norms of
the state-stationarity, input-stationarity and dynamics-feasibility residuals.  The
reference takes its ``StackedSystem``; here the ``GpuSchurOperator`` carries the same
problem data (and its ``offset`` is the stacked omega~).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import DimensionMismatchError
from .problem import GridLayout
from .solver import GpuSchurOperator, _Vec, _ptr, _torch_cuda


@dataclass
class TrajectorySolution:
    """Recovered primal trajectory plus the multipliers it came from
    (``recovery.py:24-45``)."""

    layout: GridLayout
    x_flat: np.ndarray
    u_flat: np.ndarray
    multipliers: np.ndarray
    objective_value: float

    def state(self, i, j):
        """States of subsystem (i, j) as a (T+1, n) array."""
        lay = self.layout
        x = np.asarray(self.x_flat.cpu() if _torch_cuda(self.x_flat) else self.x_flat)
        return np.stack([x[lay.x_slice(i, j, t)] for t in range(lay.T + 1)])

    def input(self, i, j):
        """Inputs of subsystem (i, j) as a (T, m) array."""
        lay = self.layout
        u = np.asarray(self.u_flat.cpu() if _torch_cuda(self.u_flat) else self.u_flat)
        return np.stack([u[lay.u_slice(i, j, t)] for t in range(lay.T)])


def _check_schur(schur):
    if not isinstance(schur, GpuSchurOperator):
        raise TypeError("expected the GpuSchurOperator that carries the problem data")


def _input_like(v, n):
    if v.device:
        import torch
        return torch.empty(n, dtype=torch.float64, device=v.obj.device)
    return np.empty(n)


def recover_solution(schur, multipliers) -> TrajectorySolution:
    """x = -Qinv (A' lam), u = -Rinv (B' lam) on the device (``recovery.py:50-65``)."""
    _check_schur(schur)
    ctx = schur._ctx
    emb = ctx.embed
    given = multipliers
    if emb is not None:      # mixed dimensions: padded vectors on the device (embed.py)
        multipliers = emb.expand_x(multipliers, "multipliers")
    lam = _Vec(multipliers, ctx.dim, "multipliers")
    nu = int(ctx.lib.gq_input_dim(ctx.h))
    x = lam.like()
    u = _input_like(lam, nu)
    obj = ctypes.c_double()
    _lib.check(ctx.lib.gq_recover(ctx.h, lam.ptr, _ptr(x), _ptr(u), ctypes.byref(obj)),
               "recover_solution")
    if emb is not None:
        return TrajectorySolution(layout=emb.layout(), x_flat=emb.restrict_x(x),
                                  u_flat=emb.restrict_u(u),
                                  multipliers=_Vec(given, schur.dim, "multipliers").obj,
                                  objective_value=float(obj.value))
    return TrajectorySolution(layout=schur.layout, x_flat=x, u_flat=u, multipliers=lam.obj,
                              objective_value=float(obj.value))


def kkt_residual(schur, sol: TrajectorySolution):
    """(||r_x||_inf, ||r_u||_inf, ||r_dyn||_inf) of ``sol`` (``recovery.py:68-80``)."""
    _check_schur(schur)
    ctx = schur._ctx
    nu = int(ctx.lib.gq_input_dim(ctx.h))
    emb = ctx.embed
    mult, xf, uf, offv = sol.multipliers, sol.x_flat, sol.u_flat, schur.offset
    if emb is not None:
        mult, xf = emb.expand_x(mult, "multipliers"), emb.expand_x(xf, "x")
        uf = emb.expand_u(uf if _torch_cuda(uf) else np.asarray(uf, dtype=float).reshape(-1), "u")
        offv = schur.arrays.offset
    lam = _Vec(mult, ctx.dim, "multipliers")
    x = _Vec(xf, ctx.dim, "x")
    if _torch_cuda(uf):
        u = _Vec(uf, nu, "u") if nu else None
    else:
        u = _Vec(np.asarray(uf, dtype=float).reshape(-1), nu, "u") if nu else None
    off = _Vec(offv, ctx.dim, "offset")
    if nu == 0:
        raise DimensionMismatchError("problem has no inputs")
    out = (ctypes.c_double * 3)()
    _lib.check(ctx.lib.gq_kkt_residual(ctx.h, lam.ptr, x.ptr, u.ptr, off.ptr,
                                       ctypes.cast(out, ctypes.c_void_p)), "kkt_residual")
    return float(out[0]), float(out[1]), float(out[2])
