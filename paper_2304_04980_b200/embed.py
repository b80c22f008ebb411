"""Heterogeneous subsystem dimensions on the uniform-n device path.

The reference's ``GridLayout`` lets every subsystem have its own state and input dimensions
(``grid_problem.py:103-170``).  The CUDA kernels are written for one block size n.  A problem
with mixed dimensions is therefore *embedded* into a uniform one:

* every state vector is padded to n_p = the smallest supported n >= max n_ij, every input
  vector to m_p = max m_ij;
* A, B and the coupling blocks are padded with zeros, Q and R with ones on the new diagonal
  entries, the initial states and boundary trajectories with zeros.

The padded states obey x+ = 0 and cost x^2 / 2, so they stay zero: Psi_t gains decoupled
identity rows (Q^-1 = 1, no Ahat or B entries), Xi_t gains zero rows, omega~ gains zeros.  The
reduced system is the reference's system plus decoupled unit equations with zero right-hand
sides; every padded multiplier is exactly zero in every PCG iterate, the padded entries add
exact zeros to every dot product and block product, and the real entries follow the same
arithmetic as an unpadded solve.  ``Embedding`` maps vectors between the reference's order
(t, j, i, k < n_ij) and the padded uniform order.
"""

from __future__ import annotations

import numpy as np

from .problem import (DIRECTIONS, BoundaryData, ConstSeq, GridLQProblem, SubsystemData)

SUPPORTED_N = (1, 2, 3, 4, 8)
MAX_M = 8


def is_heterogeneous(problem) -> bool:
    n0, m0 = problem.sub(0, 0).n, problem.sub(0, 0).m
    return any(problem.sub(i, j).n != n0 or problem.sub(i, j).m != m0
               for i in range(problem.K) for j in range(problem.N))


def needs_embedding(problem) -> bool:
    """Mixed dimensions, or a uniform state dimension the kernels are not compiled for."""
    return is_heterogeneous(problem) or problem.sub(0, 0).n not in SUPPORTED_N


def _pad_block(block, rows, cols, unit_diag):
    a = np.asarray(block, dtype=float)
    out = np.zeros((rows, cols))
    out[:a.shape[0], :a.shape[1]] = a
    if unit_diag:
        for k in range(a.shape[0], rows):
            out[k, k] = 1.0
    return out


def _pad_seq(seq, rows, cols, unit_diag=False):
    """Pad every block of a per-stage sequence; sequences that repeat one object stay so."""
    if seq is None:
        return None
    if isinstance(seq, ConstSeq):
        return ConstSeq(_pad_block(seq.obj, rows, cols, unit_diag), len(seq))
    if len(seq) and all(x is seq[0] for x in seq):
        return ConstSeq(_pad_block(seq[0], rows, cols, unit_diag), len(seq))
    return [_pad_block(b, rows, cols, unit_diag) for b in seq]


def _pad_vec(v, n):
    a = np.asarray(v, dtype=float).reshape(-1)
    out = np.zeros(n)
    out[:a.shape[0]] = a
    return out


class Embedding:
    """Index maps between a heterogeneous problem's vectors and the padded uniform ones."""

    def __init__(self, problem):
        K, N, T = problem.K, problem.N, problem.T
        self.K, self.N, self.T = K, N, T
        self.nd = np.array([[problem.sub(i, j).n for i in range(K)] for j in range(N)])  # [N][K]
        self.md = np.array([[problem.sub(i, j).m for i in range(K)] for j in range(N)])
        nmax, mmax = int(self.nd.max()), int(self.md.max())
        fits = [n for n in SUPPORTED_N if n >= nmax]
        if not fits or mmax > MAX_M:
            from .errors import DimensionMismatchError
            raise DimensionMismatchError(
                f"the B200 path supports state dimensions up to {SUPPORTED_N[-1]} and input "
                f"dimensions up to {MAX_M} (got max n={nmax}, max m={mmax})")
        self.n, self.m = fits[0], mmax
        self.x_idx = self._index(self.nd, self.n, T + 1)
        self.u_idx = self._index(self.md, self.m, T)
        self.dim = int(self.x_idx.shape[0])                 # the reference's n_total
        self.dim_pad = K * N * self.n * (T + 1)
        self.udim = int(self.u_idx.shape[0])
        self.udim_pad = K * N * self.m * T
        self._torch_idx = {}

    def _index(self, dims, width, stages):
        """Positions, in the padded (t, j, i, k < width) order, of the real entries
        (t, j, i, k < dims[j][i]) in the reference's order."""
        flat = dims.reshape(-1)                               # node order (j, i)
        node = np.repeat(np.arange(flat.shape[0]), flat)
        comp = np.concatenate([np.arange(d) for d in flat]) if flat.sum() else np.zeros(0, int)
        stage0 = node * width + comp
        per_stage = flat.shape[0] * width
        return (np.arange(stages)[:, None] * per_stage + stage0[None, :]).reshape(-1).astype(np.int64)

    # -- vectors -------------------------------------------------------------------------
    def _tidx(self, idx, device):
        import torch
        key = (id(idx), str(device))
        if key not in self._torch_idx:
            self._torch_idx[key] = torch.as_tensor(idx, device=device)
        return self._torch_idx[key]

    def _expand(self, v, idx, size, name):
        from .errors import DimensionMismatchError
        from .solver import _torch_cuda
        if _torch_cuda(v):
            import torch
            if v.dim() != 1 or v.numel() != idx.shape[0]:
                raise DimensionMismatchError(f"{name} must have length {idx.shape[0]}")
            out = torch.zeros(size, dtype=torch.float64, device=v.device)
            out[self._tidx(idx, v.device)] = v.to(torch.float64)
            return out
        a = np.asarray(v, dtype=float)
        if a.ndim != 1 or a.shape[0] != idx.shape[0]:
            raise DimensionMismatchError(
                f"{name} has shape {a.shape}, operator dimension is {idx.shape[0]}")
        out = np.zeros(size)
        out[idx] = a
        return out

    def _restrict(self, v, idx):
        from .solver import _torch_cuda
        if _torch_cuda(v):
            return v[self._tidx(idx, v.device)]
        return np.asarray(v)[idx]

    def expand_x(self, v, name="x"):
        return self._expand(v, self.x_idx, self.dim_pad, name)

    def restrict_x(self, v):
        return self._restrict(v, self.x_idx)

    def expand_u(self, v, name="u"):
        return self._expand(v, self.u_idx, self.udim_pad, name)

    def restrict_u(self, v):
        return self._restrict(v, self.u_idx)

    def layout(self):
        return HeteroLayout(self)

    # -- the padded problem --------------------------------------------------------------
    def padded_problem(self, problem) -> GridLQProblem:
        K, N, n, m = self.K, self.N, self.n, self.m
        subs = []
        for i in range(K):
            row = []
            for j in range(N):
                s = problem.sub(i, j)
                kw = {d: _pad_seq(s.coupling(d), n, n) for d in DIRECTIONS}
                row.append(SubsystemData(
                    n=n, m=m, A=_pad_seq(s.A, n, n), B=_pad_seq(s.B, n, m),
                    Q=_pad_seq(s.Q, n, n, unit_diag=True), R=_pad_seq(s.R, m, m, unit_diag=True),
                    **kw))
            subs.append(row)
        b = problem.boundary
        init = [[_pad_vec(b.init[i][j], n) for j in range(N)] for i in range(K)]

        def traj(t):
            return None if t is None else [[_pad_vec(x, n) for x in seq] for seq in t]

        bnd = BoundaryData(init=init, north=traj(b.north), south=traj(b.south),
                           west=traj(b.west), east=traj(b.east))
        return GridLQProblem(K, N, self.T, subs, bnd)


class HeteroLayout:
    """The reference's ``GridLayout`` index map for mixed dimensions
    (``grid_problem.py:103-170``): slices of the reference-order state and input vectors."""

    def __init__(self, emb: Embedding):
        self.K, self.N, self.T = emb.K, emb.N, emb.T
        self.n = [[int(emb.nd[j][i]) for j in range(emb.N)] for i in range(emb.K)]
        self.m = [[int(emb.md[j][i]) for j in range(emb.N)] for i in range(emb.K)]
        self.nhat, self.mhat = int(emb.nd.sum()), int(emb.md.sum())
        self.n_total, self.m_total = self.nhat * (emb.T + 1), self.mhat * emb.T
        self._xo = np.concatenate([[0], np.cumsum(emb.nd.reshape(-1))]).astype(int)   # (j, i)
        self._uo = np.concatenate([[0], np.cumsum(emb.md.reshape(-1))]).astype(int)
        self.pairs = [tuple(range(j, min(j + 2, self.N))) for j in range(0, self.N, 2)]

    def x_offset(self, i, j, t):
        return t * self.nhat + int(self._xo[j * self.K + i])

    def u_offset(self, i, j, t):
        return t * self.mhat + int(self._uo[j * self.K + i])

    def x_slice(self, i, j, t):
        o = self.x_offset(i, j, t)
        return slice(o, o + self.n[i][j])

    def u_slice(self, i, j, t):
        o = self.u_offset(i, j, t)
        return slice(o, o + self.m[i][j])
