"""Problem description accepted by the B200 PCGM path.

Two input forms are accepted:

* ``GridLQProblem`` -- the reference's own data model (``gridlq/grid_problem.py:29-82``):
  per-subsystem lists of per-stage matrices ``A, B, Q, R`` and the four optional
  coupling lists ``west/east/north/south``, plus ``BoundaryData`` (initial states and
  optional boundary trajectories).  The classes below mirror those fields, and any
  duck-typed object with the same attributes (e.g. a ``gridlq.GridLQProblem``) is
  accepted as well.
* ``GridArrays`` -- the dense, stage-deduplicated arrays the device consumes.  It is what
  ``GridLQProblem`` ingestion produces and what the large-scale generators emit directly
  (building 65k ``SubsystemData`` objects is pointless when every stage shares one
  matrix).

Stage deduplication ("stage classes"): for time-invariant data every stage t >= 1 has
bitwise identical Psi_t / Xi_t / pair factors, so the device
stores per-class operator data and a stage -> class map instead of T+1 copies.  A general
time-varying problem simply gets one class per stage.

Global vector order is the reference's (t, j, i, k): offset
``t*nhat + (j*K + i)*n + k`` (``grid_problem.py:143-144``), for uniform n.
"""

from __future__ import annotations

import hashlib
from collections.abc import Sequence
from dataclasses import dataclass

import numpy as np

from .errors import DimensionMismatchError, NotPositiveDefiniteError

DIRECTIONS = ("west", "east", "north", "south")
PIVOT_RTOL = 1e-14      # block_linalg.py:22
SYMMETRY_RTOL = 1e-12   # block_linalg.py:24


class ConstSeq(Sequence):
    """Read-only sequence returning the same object ``length`` times.

    Equivalent to ``[obj] * length`` for every consumer (indexing, len, iteration) but
    O(1) in memory; the generators use it so a 256x256x200 problem does not hold 100M
    list slots.  Ingestion recognises it as time-invariant without comparing stages.
    """

    __slots__ = ("obj", "length")

    def __init__(self, obj, length):
        self.obj = obj
        self.length = int(length)

    def __len__(self):
        return self.length

    def __getitem__(self, idx):
        if isinstance(idx, slice):
            return [self.obj] * len(range(*idx.indices(self.length)))
        if idx < 0:
            idx += self.length
        if not 0 <= idx < self.length:
            raise IndexError(idx)
        return self.obj


@dataclass
class SubsystemData:
    """Per-subsystem dynamics and cost data (mirror of ``grid_problem.py:29-52``)."""

    n: int
    m: int
    A: list
    B: list
    Q: list
    R: list
    west: list | None = None
    east: list | None = None
    north: list | None = None
    south: list | None = None

    def coupling(self, direction):
        return getattr(self, direction)


@dataclass
class BoundaryData:
    """Initial states and optional boundary trajectories (``grid_problem.py:55-70``)."""

    init: list
    north: list | None = None
    south: list | None = None
    west: list | None = None
    east: list | None = None


@dataclass
class GridLQProblem:
    """K x N grid of coupled subsystems over horizon T (``grid_problem.py:73-82``)."""

    K: int
    N: int
    T: int
    subsystems: list
    boundary: BoundaryData

    def sub(self, i, j) -> SubsystemData:
        return self.subsystems[i][j]


class GridLayout:
    """Uniform-n index map for the stacked multiplier vector (``grid_problem.py:103-170``).

    Stage-major, column-major inside a stage: ``x_offset(i,j,t) = t*nhat + (j*K+i)*n``.
    Column pairs ``[(0,1),(2,3),...]`` with a singleton last pair for odd N (``:135-137``).
    """

    def __init__(self, K, N, T, n, m=0):
        self.K, self.N, self.T, self.n, self.m = int(K), int(N), int(T), int(n), int(m)
        self.nhat = self.K * self.N * self.n
        self.mhat = self.K * self.N * self.m
        self.n_total = self.nhat * (self.T + 1)
        self.m_total = self.mhat * self.T
        self.pairs = [tuple(range(j, min(j + 2, self.N))) for j in range(0, self.N, 2)]

    @property
    def n_pairs(self):
        return len(self.pairs)

    def x_offset(self, i, j, t):
        return t * self.nhat + (j * self.K + i) * self.n

    def x_slice(self, i, j, t):
        o = self.x_offset(i, j, t)
        return slice(o, o + self.n)

    def stage_x_slice(self, t):
        return slice(t * self.nhat, (t + 1) * self.nhat)

    def u_offset(self, i, j, t):
        """Input vector order (``grid_problem.py:146-161``): ``t*mhat + (j*K+i)*m``."""
        return t * self.mhat + (j * self.K + i) * self.m

    def u_slice(self, i, j, t):
        o = self.u_offset(i, j, t)
        return slice(o, o + self.m)

    def stage_u_slice(self, t):
        return slice(t * self.mhat, (t + 1) * self.mhat)


@dataclass
class GridArrays:
    """Dense, stage-class-deduplicated problem data (host numpy, float64).

    Node axes are ordered ``[N][K]`` (column j, then row i) to match the in-stage vector
    order.  ``dyn_class[t]`` (t < T) selects the dynamics set (A, B, R, couplings) used
    between stages t and t+1; ``cost_class[t]`` (t <= T) selects the state-cost set Q_t.

    * ``A``  [n_dyn, N, K, n, n]
    * ``B``  [n_dyn, N, K, n, m]
    * ``R``  [n_dyn, N, K, m, m]
    * ``C``  [n_dyn, 4, N, K, n, n]  in-grid couplings (west, east, north, south); zeros
      where the subsystem declares none
    * ``cmask`` [4, N, K] bool -- coupling list declared (not None); only the reference's
      stored-block bookkeeping (flop counters) depends on it
    * ``Q``  [n_cost, N, K, n, n]
    * ``offset`` [dim] -- the reduced right-hand side omega~ (``kkt_assembly.py:275-301``)
    """

    K: int
    N: int
    T: int
    n: int
    m: int
    A: np.ndarray
    B: np.ndarray
    R: np.ndarray
    C: np.ndarray
    cmask: np.ndarray
    Q: np.ndarray
    dyn_class: np.ndarray
    cost_class: np.ndarray
    offset: np.ndarray

    @property
    def dim(self):
        return self.K * self.N * self.n * (self.T + 1)

    @property
    def layout(self):
        return GridLayout(self.K, self.N, self.T, self.n, self.m)

    @property
    def time_invariant(self):
        return len(self.A) == 1 and len(self.Q) == 1

    def psi_classes(self):
        """Stage -> Psi class map and the class keys.

        Psi_0 = Qinv_0; Psi_t (t>=1) = Qinv_t + Ahat_{t-1} Qinv_{t-1} Ahat_{t-1}' +
        B R^-1 B' (``kkt_assembly.py:493-533``), so its data key is
        (cost_class[t], dyn_class[t-1], cost_class[t-1]); key dyn = -1 marks stage 0.
        """
        keys, cls = {}, np.empty(self.T + 1, dtype=np.int32)
        for t in range(self.T + 1):
            if t == 0:
                key = (int(self.cost_class[0]), -1, -1)
            else:
                key = (int(self.cost_class[t]), int(self.dyn_class[t - 1]),
                       int(self.cost_class[t - 1]))
            cls[t] = keys.setdefault(key, len(keys))
        return cls, np.array(list(keys), dtype=np.int32).reshape(-1, 3)

    def xi_classes(self):
        """Stage -> Xi class map; Xi_t = -Ahat_t Qinv_t (``kkt_assembly.py:535-543``)."""
        keys, cls = {}, np.empty(self.T, dtype=np.int32)
        for t in range(self.T):
            key = (int(self.dyn_class[t]), int(self.cost_class[t]))
            cls[t] = keys.setdefault(key, len(keys))
        return cls, np.array(list(keys), dtype=np.int32).reshape(-1, 2)


# ---------------------------------------------------------------------------
# validation (semantics of grid_problem.py:181-288, raised as build_stacked does)


def _cholesky_ok(mats):
    """Batched check that every matrix passes the reference's dense_cholesky
    (``block_linalg.py:43-65``): symmetric within 1e-12 and pivots above
    PIVOT_RTOL * max diag."""
    mats = np.asarray(mats, dtype=float)
    if mats.size == 0:
        return np.ones(mats.shape[:-2], dtype=bool)
    scale = np.maximum(1.0, np.max(np.abs(mats), axis=(-1, -2)))
    sym = np.max(np.abs(mats - np.swapaxes(mats, -1, -2)), axis=(-1, -2)) / scale <= SYMMETRY_RTOL
    n = mats.shape[-1]
    lower = np.zeros_like(mats)
    tol = PIVOT_RTOL * np.max(np.diagonal(mats, axis1=-2, axis2=-1), axis=-1)
    ok = sym.copy()
    for j in range(n):
        piv = mats[..., j, j] - np.sum(lower[..., j, :j] ** 2, axis=-1)
        ok &= piv > tol
        ljj = np.sqrt(np.where(piv > 0, piv, 1.0))
        lower[..., j, j] = ljj
        if j + 1 < n:
            lower[..., j + 1:, j] = (
                mats[..., j + 1:, j] - np.einsum("...rk,...k->...r", lower[..., j + 1:, :j],
                                                 lower[..., j, :j])
            ) / ljj[..., None]
    return ok


def validate_arrays(ga: GridArrays) -> list:
    """Invariant violations of a GridArrays instance; empty means valid."""
    msgs = []
    if ga.K < 1 or ga.N < 1 or ga.T < 1:
        return [f"grid dimensions must be positive, got K={ga.K} N={ga.N} T={ga.T}"]
    if ga.n < 1 or ga.m < 1:
        return [f"dimensions n={ga.n} m={ga.m} must be positive"]
    nd, nq = len(ga.A), len(ga.Q)
    shapes = {
        "A": (ga.A, (nd, ga.N, ga.K, ga.n, ga.n)),
        "B": (ga.B, (nd, ga.N, ga.K, ga.n, ga.m)),
        "R": (ga.R, (nd, ga.N, ga.K, ga.m, ga.m)),
        "C": (ga.C, (nd, 4, ga.N, ga.K, ga.n, ga.n)),
        "Q": (ga.Q, (nq, ga.N, ga.K, ga.n, ga.n)),
    }
    for name, (arr, want) in shapes.items():
        if tuple(arr.shape) != want:
            msgs.append(f"{name}: shape {tuple(arr.shape)}, expected {want}")
    if msgs:
        return msgs
    if len(ga.dyn_class) != ga.T or len(ga.cost_class) != ga.T + 1:
        msgs.append("stage class maps do not match T")
    if np.any(ga.dyn_class < 0) or np.any(ga.dyn_class >= nd):
        msgs.append("dyn_class out of range")
    if np.any(ga.cost_class < 0) or np.any(ga.cost_class >= nq):
        msgs.append("cost_class out of range")
    if ga.offset.shape != (ga.dim,):
        msgs.append(f"offset has shape {ga.offset.shape}, expected {(ga.dim,)}")
    for name, arr in (("Q", ga.Q), ("R", ga.R)):
        ok = _cholesky_ok(arr)
        if not np.all(ok):
            c, j, i = np.argwhere(~ok)[0]
            msgs.append(f"subsystem ({i}, {j}): {name} (set {c}): not symmetric positive definite")
    for arr_name in ("A", "B", "R", "C", "Q", "offset"):
        if not np.all(np.isfinite(getattr(ga, arr_name))):
            msgs.append(f"{arr_name} contains non-finite entries")
    return msgs


# ---------------------------------------------------------------------------
# GridLQProblem -> GridArrays


def _is_const(seq):
    if isinstance(seq, ConstSeq):
        return True
    if len(seq) == 0:
        return True
    first = seq[0]
    if all(x is first for x in seq):
        return True
    a0 = np.asarray(first, dtype=float)
    return all(np.array_equal(np.asarray(x, dtype=float), a0) for x in seq)


def _stage_ids(K, N, seq_at, count, shape):
    """Per-stage ids for one field: stages holding identical data for every node share
    an id.  ``seq_at(i, j)`` returns that node's per-stage sequence or None.  Returns
    (ids[count], per-id stacked arrays [n_ids, N, K, *shape]).

    Vectorised: each node's sequence is converted with ONE ``np.asarray`` (a C loop over
    its stages) into a dense [count, N, K, *shape] array, and equal stages are found with
    one ``np.unique`` over the stage rows -- O(K N) Python calls instead of O(T K N)."""
    seqs = [[seq_at(i, j) for i in range(K)] for j in range(N)]
    if all(_is_const(s) for col in seqs for s in col if s is not None):
        ids = np.zeros(count, dtype=np.int32)
        stack = np.zeros((1, N, K) + shape)
        for j in range(N):
            for i in range(K):
                s = seqs[j][i]
                if s is not None and len(s):
                    stack[0, j, i] = np.asarray(s[0], dtype=float)
        return ids, stack
    dense = np.zeros((N, K, count) + shape)
    for j in range(N):
        for i in range(K):
            s = seqs[j][i]
            if s is not None:
                dense[j, i] = np.asarray(s if not isinstance(s, ConstSeq) else [s[0]] * count,
                                         dtype=float).reshape((count,) + shape)
    per_t = np.ascontiguousarray(np.moveaxis(dense, 2, 0))          # [count, N, K, *shape]
    rows = per_t.reshape(count, -1).view(np.uint8).reshape(count, -1)
    _, first, inv = np.unique(rows, axis=0, return_index=True, return_inverse=True)
    # ids numbered by first appearance (the order the stage loop would assign them)
    order = np.argsort(first, kind="stable")
    rank = np.empty_like(order)
    rank[order] = np.arange(len(order))
    ids = rank[inv.reshape(-1)].astype(np.int32)
    return ids, per_t[np.sort(first)]


_NEIGHBOR = {"west": (0, -1), "east": (0, 1), "north": (-1, 0), "south": (1, 0)}


def _problem_messages(problem):
    """Structural checks of grid_problem.validate (``grid_problem.py:195-288``) that the
    dense conversion relies on."""
    msgs = []
    K, N, T = problem.K, problem.N, problem.T
    if K < 1 or N < 1 or T < 1:
        return [f"grid dimensions must be positive, got K={K} N={N} T={T}"]
    if len(problem.subsystems) != K or any(len(r) != N for r in problem.subsystems):
        return ["subsystem table does not match K x N"]
    for i in range(K):
        for j in range(N):
            sub = problem.sub(i, j)
            tag = f"subsystem ({i}, {j})"
            n, m = sub.n, sub.m
            if n < 1 or m < 1:
                msgs.append(f"{tag}: dimensions n={n} m={m} must be positive")
                continue
            for name, seq, cnt, shape in (("A", sub.A, T, (n, n)), ("B", sub.B, T, (n, m)),
                                          ("Q", sub.Q, T + 1, (n, n)), ("R", sub.R, T, (m, m))):
                if len(seq) != cnt:
                    msgs.append(f"{tag}: {name} has {len(seq)} stages, expected {cnt}")
                    continue
                probe = [seq[0]] if isinstance(seq, ConstSeq) else seq
                for t, mat in enumerate(probe):
                    if np.asarray(mat).shape != shape:
                        msgs.append(f"{tag}: {name}[{t}] shape {np.asarray(mat).shape}, expected {shape}")
                        break
            for direction in DIRECTIONS:
                blocks = sub.coupling(direction)
                if blocks is None:
                    continue
                if len(blocks) != T:
                    msgs.append(f"{tag}: {direction} coupling has {len(blocks)} stages, expected {T}")
                    continue
                ni, nj = {"west": (i, j - 1), "east": (i, j + 1), "north": (i - 1, j),
                          "south": (i + 1, j)}[direction]
                if 0 <= ni < K and 0 <= nj < N:
                    want = problem.sub(ni, nj).n
                else:
                    traj = getattr(problem.boundary, direction)
                    if traj is None:
                        msgs.append(f"{tag}: {direction} coupling points off-grid but no "
                                    "boundary trajectory is declared")
                        continue
                    want = len(np.asarray(traj[j if direction in ("north", "south") else i][0]))
                probe = [blocks[0]] if isinstance(blocks, ConstSeq) else blocks
                for t, blk in enumerate(probe):
                    if np.asarray(blk).shape != (n, want):
                        msgs.append(f"{tag}: {direction} coupling[{t}] shape "
                                    f"{np.asarray(blk).shape}, expected {(n, want)}")
                        break
    init = problem.boundary.init
    if len(init) != K or any(len(r) != N for r in init):
        msgs.append("boundary.init does not match K x N")
    else:
        for i in range(K):
            for j in range(N):
                if np.asarray(init[i][j]).shape != (problem.sub(i, j).n,):
                    msgs.append(f"initial state ({i}, {j}): shape "
                                f"{np.asarray(init[i][j]).shape}, expected {(problem.sub(i, j).n,)}")
    for direction, count in (("north", N), ("south", N), ("west", K), ("east", K)):
        traj = getattr(problem.boundary, direction)
        if traj is None:
            continue
        if len(traj) != count:
            msgs.append(f"boundary.{direction} has {len(traj)} entries, expected {count}")
            continue
        for idx, seq in enumerate(traj):
            if len(seq) != T:
                msgs.append(f"boundary.{direction}[{idx}] has {len(seq)} stages, expected {T}")
    return msgs


def arrays_from_problem(problem) -> GridArrays:
    """Convert a (reference-shaped) GridLQProblem into GridArrays.

    Raises ValueError for invalid problems exactly where ``build_stacked`` would
    (``kkt_assembly.py:209-211``) and DimensionMismatchError for heterogeneous
    state/input dimensions, which the B200 path does not support.
    """
    msgs = _problem_messages(problem)
    if msgs:
        raise ValueError("invalid problem: " + "; ".join(msgs))
    K, N, T = problem.K, problem.N, problem.T
    n, m = problem.sub(0, 0).n, problem.sub(0, 0).m
    for i in range(K):
        for j in range(N):
            s = problem.sub(i, j)
            if s.n != n or s.m != m:
                raise DimensionMismatchError(
                    "GridArrays hold one block size: mixed dimensions go through "
                    "GpuSchurOperator(problem), which embeds them (embed.py) "
                    f"(got n={s.n}, m={s.m} at ({i}, {j}) vs n={n}, m={m})")
    ids = {}
    stacks = {}
    ids["A"], stacks["A"] = _stage_ids(K, N, lambda i, j: problem.sub(i, j).A, T, (n, n))
    ids["B"], stacks["B"] = _stage_ids(K, N, lambda i, j: problem.sub(i, j).B, T, (n, m))
    ids["R"], stacks["R"] = _stage_ids(K, N, lambda i, j: problem.sub(i, j).R, T, (m, m))
    ids["Q"], stacks["Q"] = _stage_ids(K, N, lambda i, j: problem.sub(i, j).Q, T + 1, (n, n))
    cmask = np.zeros((4, N, K), dtype=bool)
    for d, direction in enumerate(DIRECTIONS):
        di, dj = _NEIGHBOR[direction]
        for j in range(N):
            for i in range(K):
                in_grid = 0 <= i + di < K and 0 <= j + dj < N
                cmask[d, j, i] = in_grid and problem.sub(i, j).coupling(direction) is not None

        # only in-grid couplings enter Ahat; off-grid ones only touch the offset
        def seq_at(i, j, d=d, direction=direction):
            return problem.sub(i, j).coupling(direction) if cmask[d, j, i] else None

        ids[direction], stacks[direction] = _stage_ids(K, N, seq_at, T, (n, n))
    keys = list(zip(*(ids[f] for f in ("A", "B", "R") + DIRECTIONS)))
    dyn_map, dyn_class = {}, np.empty(T, dtype=np.int32)
    for t, key in enumerate(keys):
        dyn_class[t] = dyn_map.setdefault(key, len(dyn_map))
    nd = len(dyn_map)
    A = np.empty((nd, N, K, n, n))
    B = np.empty((nd, N, K, n, m))
    R = np.empty((nd, N, K, m, m))
    C = np.empty((nd, 4, N, K, n, n))
    for key, c in dyn_map.items():
        A[c] = stacks["A"][key[0]]
        B[c] = stacks["B"][key[1]]
        R[c] = stacks["R"][key[2]]
        for d, direction in enumerate(DIRECTIONS):
            C[c, d] = stacks[direction][key[3 + d]]
    offset = rhs_offset(problem, n)
    ga = GridArrays(K, N, T, n, m, A, B, R, C, cmask, stacks["Q"], dyn_class,
                    ids["Q"].astype(np.int32), offset)
    msgs = validate_arrays(ga)
    if msgs:
        raise ValueError("invalid problem: " + "; ".join(msgs))
    return ga


def rhs_offset(problem, n):
    """omega~: initial states at stage 0 plus boundary-trajectory terms at stage t+1
    (``kkt_assembly.py:275-301``).  Vectorised over stages: per edge node and direction
    the T coupling blocks and trajectory samples are stacked once and applied as one
    batched product (``np.einsum``), not T separate matrix-vector products."""
    K, N, T = problem.K, problem.N, problem.T
    nk = K * N * n
    offset = np.zeros((T + 1) * nk)
    bnd = problem.boundary
    init = np.asarray(bnd.init, dtype=float).reshape(K, N, n)        # [i][j][k]
    offset[:nk] = np.transpose(init, (1, 0, 2)).reshape(-1)          # order (j, i, k)
    if all(getattr(bnd, d) is None for d in DIRECTIONS):
        return offset
    stages = offset[nk:].reshape(T, N, K, n)                         # stages 1..T
    for direction in ("north", "south", "west", "east"):
        traj = getattr(bnd, direction)
        if traj is None:
            continue
        if direction in ("north", "south"):
            i = 0 if direction == "north" else K - 1
            nodes = [(i, j, j) for j in range(N)]
        else:
            j = 0 if direction == "west" else N - 1
            nodes = [(i, j, i) for i in range(K)]
        for i, j, idx in nodes:
            blocks = problem.sub(i, j).coupling(direction)
            if blocks is None:
                continue
            Cs = np.asarray(blocks, dtype=float).reshape(T, n, n)
            sig = np.asarray(traj[idx], dtype=float).reshape(T, n)
            stages[:, j, i] += np.einsum("tab,tb->ta", Cs, sig)
    return offset


def boundary_arrays(problem, n):
    """The inputs of ``gq_build_offset`` as dense host arrays: ``init`` [N][K][n], the edge
    coupling ``blocks`` [4][L][ncls][n][n] (L = max(K, N); direction order DIRECTIONS), their
    stage ``cls`` map [4][L][T] (-1: no coupling list or no trajectory -> no term) and the
    boundary trajectories ``traj`` [4][L][T][n].  A coupling list that repeats one block
    (``ConstSeq``) is one class; any other list keeps its T blocks."""
    K, N, T = problem.K, problem.N, problem.T
    L = max(K, N)
    bnd = problem.boundary
    init = np.ascontiguousarray(
        np.transpose(np.asarray(bnd.init, dtype=float).reshape(K, N, n), (1, 0, 2)))
    edges = {}
    varying = False
    for d, direction in enumerate(DIRECTIONS):
        traj = getattr(bnd, direction)
        if traj is None:
            continue
        if direction in ("north", "south"):
            i = 0 if direction == "north" else K - 1
            nodes = [(i, j, j) for j in range(N)]
        else:
            j = 0 if direction == "west" else N - 1
            nodes = [(i, j, i) for i in range(K)]
        for i, j, e in nodes:
            blocks = problem.sub(i, j).coupling(direction)
            if blocks is None:
                continue
            const = isinstance(blocks, ConstSeq)
            varying = varying or not const
            edges[(d, e)] = (blocks, const, traj[e])
    ncls = T if varying else 1
    blk = np.zeros((4, L, ncls, n, n))
    cls = np.full((4, L, T), -1, dtype=np.int32)
    tr = np.zeros((4, L, T, n))
    for (d, e), (blocks, const, sig) in edges.items():
        if const:
            blk[d, e, 0] = np.asarray(blocks[0], dtype=float)
            cls[d, e] = 0
        else:
            blk[d, e] = np.asarray(blocks, dtype=float).reshape(T, n, n)
            cls[d, e] = np.arange(T)
        tr[d, e] = np.asarray(sig, dtype=float).reshape(T, n)
    return init, blk, cls, tr


def rhs_offset_device(problem, n=None, device="cuda"):
    """omega~ (``kkt_assembly.py:275-301``) as a CUDA tensor in the reference vector order,
    built by the ``gq_build_offset`` kernel from the boundary data: the device-side
    counterpart of ``rhs_offset`` for right-hand sides that never need to exist on the host."""
    import ctypes

    import torch

    from . import _lib

    if n is None:
        n = problem.sub(0, 0).n
    K, N, T = problem.K, problem.N, problem.T
    init, blk, cls, tr = boundary_arrays(problem, n)
    dev = [torch.as_tensor(a, device=device) for a in (init, blk, cls, tr)]
    out = torch.empty((T + 1) * K * N * n, dtype=torch.float64, device=device)
    stream = torch.cuda.current_stream(out.device).cuda_stream
    with torch.cuda.device(out.device):
        _lib.check(_lib.load().gq_build_offset(
            K, N, T, n, blk.shape[2], *(ctypes.c_void_p(t.data_ptr()) for t in dev),
            ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(stream)), "gq_build_offset")
    return out


def problem_messages(problem):
    """The reference's ``validate`` messages for a problem (``grid_problem.py:195-288``)."""
    return _problem_messages(problem)


def as_arrays(problem_or_arrays) -> GridArrays:
    if isinstance(problem_or_arrays, GridArrays):
        msgs = validate_arrays(problem_or_arrays)
        if msgs:
            raise ValueError("invalid problem: " + "; ".join(msgs))
        return problem_or_arrays
    return arrays_from_problem(problem_or_arrays)


def arrays_to_problem(ga: GridArrays, boundary: BoundaryData | None = None) -> GridLQProblem:
    """Rebuild a GridLQProblem view of GridArrays (ConstSeq lists for time-invariant
    fields).  Used to feed the reference/oracle the byte-identical problem."""
    K, N, T = ga.K, ga.N, ga.T
    ti_dyn = np.all(ga.dyn_class == ga.dyn_class[0])
    ti_q = np.all(ga.cost_class == ga.cost_class[0])

    def seq(getter, classes, count):
        if np.all(classes == classes[0]):
            return ConstSeq(getter(int(classes[0])), count)
        cache = {}
        return [cache.setdefault(int(c), getter(int(c))) for c in classes]

    subs = []
    for i in range(K):
        row = []
        for j in range(N):
            kw = {}
            for d, direction in enumerate(DIRECTIONS):
                if ga.cmask[d, j, i]:
                    kw[direction] = seq(lambda c, d=d: ga.C[c, d, j, i], ga.dyn_class, T)
            row.append(SubsystemData(
                n=ga.n, m=ga.m,
                A=seq(lambda c: ga.A[c, j, i], ga.dyn_class, T),
                B=seq(lambda c: ga.B[c, j, i], ga.dyn_class, T),
                Q=seq(lambda c: ga.Q[c, j, i], ga.cost_class, T + 1),
                R=seq(lambda c: ga.R[c, j, i], ga.dyn_class, T),
                **kw))
        subs.append(row)
    del ti_dyn, ti_q
    if boundary is None:
        lay = ga.layout
        init = [[ga.offset[lay.x_slice(i, j, 0)].copy() for j in range(N)] for i in range(K)]
        boundary = BoundaryData(init=init)
    return GridLQProblem(K, N, T, subs, boundary)


def check_spd_blocks(mats, what):
    ok = _cholesky_ok(mats)
    if not np.all(ok):
        raise NotPositiveDefiniteError(f"{what}: not positive definite")


# ---- problem files (JSON, ``grid_problem.py:431-529``) --------------------------------------
# Same self-describing document as the reference ("format": "grid-lq-problem", version 1);
# floats go through repr, so load(save(p)) reproduces every matrix bit for bit.

def _mats_to_lists(seq):
    if seq is None:
        return None
    return [np.asarray(m).tolist() for m in seq]


def _lists_to_mats(seq):
    if seq is None:
        return None
    return [np.array(m, dtype=float) for m in seq]


def problem_to_dict(problem) -> dict:
    """``grid_problem.py:444-476``"""
    subs = []
    for i in range(problem.K):
        row = []
        for j in range(problem.N):
            s = problem.sub(i, j)
            row.append({"n": s.n, "m": s.m, "A": _mats_to_lists(s.A), "B": _mats_to_lists(s.B),
                        "Q": _mats_to_lists(s.Q), "R": _mats_to_lists(s.R),
                        **{d: _mats_to_lists(s.coupling(d)) for d in DIRECTIONS}})
        subs.append(row)
    bnd = problem.boundary
    return {
        "format": "grid-lq-problem",
        "version": 1,
        "K": problem.K,
        "N": problem.N,
        "T": problem.T,
        "subsystems": subs,
        "boundary": {
            "init": [[np.asarray(g).tolist() for g in row] for row in bnd.init],
            **{d: None if getattr(bnd, d) is None
               else [[np.asarray(v).tolist() for v in seq] for seq in getattr(bnd, d)]
               for d in DIRECTIONS},
        },
    }


def problem_from_dict(data: dict) -> GridLQProblem:
    """``grid_problem.py:479-510``; ValueError for a document of another format."""
    if data.get("format") != "grid-lq-problem":
        raise ValueError("not a grid-lq-problem document")
    subs = []
    for row in data["subsystems"]:
        subs.append([SubsystemData(n=int(rec["n"]), m=int(rec["m"]), A=_lists_to_mats(rec["A"]),
                                   B=_lists_to_mats(rec["B"]), Q=_lists_to_mats(rec["Q"]),
                                   R=_lists_to_mats(rec["R"]),
                                   **{d: _lists_to_mats(rec.get(d)) for d in DIRECTIONS})
                     for rec in row])
    bnd = data["boundary"]
    boundary = BoundaryData(
        init=[[np.array(g, dtype=float) for g in row] for row in bnd["init"]],
        **{d: None if bnd.get(d) is None
           else [[np.array(v, dtype=float) for v in seq] for seq in bnd[d]]
           for d in DIRECTIONS})
    return GridLQProblem(int(data["K"]), int(data["N"]), int(data["T"]), subs, boundary)


def save_problem(problem, path):
    """``grid_problem.py:513-523``"""
    import json

    with open(path, "w") as fh:
        json.dump(problem_to_dict(problem), fh)
        fh.write("\n")


def load_problem(path) -> GridLQProblem:
    """``grid_problem.py:526-529``"""
    import json

    with open(path) as fh:
        return problem_from_dict(json.load(fh))
