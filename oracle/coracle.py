"""ctypes front-end of oracle/gridlq_oracle.c -- TEST INFRASTRUCTURE ONLY.

``COracle(Oracle)`` reuses the numpy oracle's setup (Psi/Xi blocks, pair factors) and
runs the per-step algorithm in C with OpenMP: the fast CPU oracle used by the bench's
CPU baseline / ``--impl reference`` leg and by large-size parity checks.  Pinned by
``tests/test_oracle_golden.py`` against the reference's golden vectors like the numpy
restatement.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "gridlq_oracle.c")
LIB = os.path.join(HERE, "_oracle_c.so")


def build(force=False):
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.run(["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-fPIC", "-shared", SRC,
                        "-o", LIB, "-lm"], check=True)
    return LIB


class _Orc(ctypes.Structure):
    _fields_ = [("K", ctypes.c_int), ("N", ctypes.c_int), ("T", ctypes.c_int),
                ("n", ctypes.c_int), ("V", ctypes.c_int), ("nb", ctypes.c_int),
                ("q", ctypes.c_int),
                ("psi_cls", ctypes.c_void_p), ("xi_cls", ctypes.c_void_p),
                ("psi", ctypes.c_void_p), ("xi", ctypes.c_void_p), ("xit", ctypes.c_void_p),
                ("linv", ctypes.c_void_p), ("sub", ctypes.c_void_p)]


_lib = None


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        vp = ctypes.c_void_p
        for name in ("orc_delta", "orc_outer", "orc_inner", "orc_pair_solve"):
            getattr(_lib, name).argtypes = [vp, vp, vp]
            getattr(_lib, name).restype = None
        _lib.orc_precond.argtypes = [vp, ctypes.c_int, ctypes.c_int, vp, vp, vp]
        _lib.orc_precond.restype = None
        _lib.orc_pcg.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, ctypes.c_double,
                                 ctypes.c_long, vp, vp, ctypes.POINTER(ctypes.c_long),
                                 ctypes.POINTER(ctypes.c_int), vp, vp]
        _lib.orc_pcg.restype = ctypes.c_int
        _lib.orc_threads.restype = ctypes.c_int
        _lib.orc_set_threads.argtypes = [ctypes.c_int]
    return _lib


class COracle:
    def __init__(self, orc, threads=None):
        lib = _load()
        if threads:
            lib.orc_set_threads(int(threads))
        self.threads = lib.orc_threads()
        self.o = orc
        self.dim = orc.dim
        self.L, self.S = orc.L, orc.S
        keep = dict(
            psi_cls=np.ascontiguousarray(orc.psi_cls, dtype=np.int32),
            xi_cls=np.ascontiguousarray(orc.xi_cls if orc.T else np.zeros(1), dtype=np.int32),
            psi=np.ascontiguousarray(np.stack(orc.psi)),
            xi=np.ascontiguousarray(np.stack(orc.xi)),
            xit=np.ascontiguousarray(np.stack(orc.xit)),
            linv=np.ascontiguousarray(np.stack([f[0] for f in orc.factors])),
            sub=np.ascontiguousarray(np.stack([f[1] for f in orc.factors])),
        )
        self._keep = keep
        self.s = _Orc(orc.K, orc.N, orc.T, orc.n, orc.V, orc.nb, orc.q,
                      *(keep[k].ctypes.data for k in ("psi_cls", "xi_cls", "psi", "xi", "xit",
                                                      "linv", "sub")))
        self.lib = lib

    def _unary(self, fn, x):
        x = np.ascontiguousarray(x, dtype=float)
        y = np.empty_like(x)
        getattr(self.lib, fn)(ctypes.byref(self.s), x.ctypes.data, y.ctypes.data)
        return y

    def apply_delta(self, x):
        return self._unary("orc_delta", x)

    def apply_outer(self, x):
        return self._unary("orc_outer", x)

    def apply_inner(self, x):
        return self._unary("orc_inner", x)

    def pair_solve(self, x):
        return self._unary("orc_pair_solve", x)

    def apply_precond(self, r):
        if self.L % 2:
            raise ValueError("preconditioner use requires an even inner budget "
                             f"(got {self.L}); odd budgets are standalone-only")
        r = np.ascontiguousarray(r, dtype=float)
        q = np.empty_like(r)
        work = np.empty(4 * self.dim)
        self.lib.orc_precond(ctypes.byref(self.s), self.L, self.S, r.ctypes.data, q.ctypes.data,
                             work.ctypes.data)
        return q

    def pcg(self, rhs, tol=1e-9, max_steps=None, precond=True):
        """Returns (x, history, steps, converged, status, cumulative step seconds)."""
        if max_steps is None:
            max_steps = self.dim + 50
        rhs = np.ascontiguousarray(rhs, dtype=float)
        x = np.empty(self.dim)
        hist = np.empty(max_steps)
        secs = np.empty(max_steps)
        work = np.empty(8 * self.dim)
        steps = ctypes.c_long()
        conv = ctypes.c_int()
        rc = self.lib.orc_pcg(ctypes.byref(self.s), self.L, self.S, int(precond), rhs.ctypes.data,
                              float(tol), int(max_steps), x.ctypes.data, hist.ctypes.data,
                              ctypes.byref(steps), ctypes.byref(conv), work.ctypes.data,
                              secs.ctypes.data)
        k = steps.value
        status = "breakdown" if rc == 2 else ("ok" if conv.value else "max_steps")
        return x, list(hist[:k]), k, bool(conv.value), status, secs[:k]
