"""Problem builders for parity cases (pure numpy; no reference import).

Besides the BASELINE.json generators these cover the edge cases the reference's own
tests exercise (``pkg/tests/conftest.py:14-97``): an uncoupled problem whose reduced
operator is the identity, the scalar chain, all four boundary trajectories, plus
ragged grids, time-varying data, a distinct terminal weight and partially missing
couplings.  Each returns a ``GridLQProblem`` built from the package's mirror classes.
"""

from __future__ import annotations

import numpy as np

from paper_2304_04980_b200.problem import BoundaryData, GridLQProblem, SubsystemData


def uncoupled(K=1, N=2, T=1, n=2, m=1, a_scale=0.0, init_scale=1.0):
    """No spatial coupling; a_scale=0 gives Delta = I (B = 0, Q = I)."""
    subs, init = [], []
    for i in range(K):
        row, irow = [], []
        for j in range(N):
            a = a_scale * np.eye(n)
            b = np.zeros((n, m)) if a_scale == 0.0 else 0.1 * np.ones((n, m))
            row.append(SubsystemData(n=n, m=m, A=[a] * T, B=[b] * T,
                                     Q=[np.eye(n)] * (T + 1), R=[np.eye(m)] * T))
            irow.append(init_scale * np.ones(n))
        subs.append(row)
        init.append(irow)
    return GridLQProblem(K, N, T, subs, BoundaryData(init=init))


def scalar_chain(a=0.7, b=0.5, q=2.0, r=3.0, T=3):
    sub = SubsystemData(n=1, m=1, A=[np.array([[a]])] * T, B=[np.array([[b]])] * T,
                        Q=[np.array([[q]])] * (T + 1), R=[np.array([[r]])] * T)
    return GridLQProblem(1, 1, T, [[sub]], BoundaryData(init=[[np.array([1.0])]]))


def boundary_problem(K=3, N=3, T=3, seed=42):
    """Couplings on every side, boundary trajectories on all four edges."""
    rng = np.random.default_rng(seed)
    n, m = 2, 1
    couple = 0.05 * np.eye(n)
    subs, init = [], []
    for i in range(K):
        row, irow = [], []
        for j in range(N):
            a = np.eye(n) + 0.1 * rng.uniform(-0.5, 0.5, (n, n))
            row.append(SubsystemData(
                n=n, m=m, A=[a] * T, B=[0.1 * np.ones((n, m))] * T,
                Q=[np.eye(n)] * (T + 1), R=[np.eye(m)] * T,
                west=[couple] * T, east=[couple] * T, north=[couple] * T, south=[couple] * T))
            irow.append(rng.uniform(-1, 1, n))
        subs.append(row)
        init.append(irow)
    bnd = BoundaryData(
        init=init,
        north=[[rng.uniform(-1, 1, n) for _ in range(T)] for _ in range(N)],
        south=[[rng.uniform(-1, 1, n) for _ in range(T)] for _ in range(N)],
        west=[[rng.uniform(-1, 1, n) for _ in range(T)] for _ in range(K)],
        east=[[rng.uniform(-1, 1, n) for _ in range(T)] for _ in range(K)])
    return GridLQProblem(K, N, T, subs, bnd)


def time_varying(K=4, N=3, T=5, n=2, m=1, seed=7, terminal_scale=3.0):
    """Every stage has its own A/B/coupling data, and Q_T differs from Q_t."""
    rng = np.random.default_rng(seed)
    subs, init = [], []
    for i in range(K):
        row, irow = [], []
        for j in range(N):
            A = [0.5 * rng.standard_normal((n, n)) for _ in range(T)]
            B = [rng.standard_normal((n, m)) for _ in range(T)]
            Q = []
            for t in range(T + 1):
                g = rng.standard_normal((n, n))
                Q.append(g @ g.T + n * np.eye(n))
            Q[-1] = terminal_scale * Q[-1]
            R = [np.eye(m) * (1.0 + t) for t in range(T)]
            kw = {}
            for d, (di, dj) in (("west", (0, -1)), ("east", (0, 1)),
                                ("north", (-1, 0)), ("south", (1, 0))):
                if 0 <= i + di < K and 0 <= j + dj < N:
                    kw[d] = [0.05 * rng.standard_normal((n, n)) for _ in range(T)]
            row.append(SubsystemData(n=n, m=m, A=A, B=B, Q=Q, R=R, **kw))
            irow.append(rng.standard_normal(n))
        subs.append(row)
        init.append(irow)
    return GridLQProblem(K, N, T, subs, BoundaryData(init=init))


def sparse_couplings(K=5, N=5, T=4, n=2, m=1, seed=11):
    """Only some subsystems declare couplings; one column's west couplings are all
    zero (the reference then stores no west piece for it, which the flop counters see)."""
    rng = np.random.default_rng(seed)
    subs, init = [], []
    for i in range(K):
        row, irow = [], []
        for j in range(N):
            a = 0.9 * np.eye(n) + 0.05 * rng.standard_normal((n, n))
            kw = {}
            if j > 0 and (i + j) % 2 == 0:
                kw["west"] = [0.0 * np.eye(n) if j == 2 else 0.1 * rng.standard_normal((n, n))] * T
            if i > 0 and j % 3 != 1:
                kw["north"] = [0.1 * rng.standard_normal((n, n))] * T
            if i < K - 1 and j != 3:
                kw["south"] = [0.1 * rng.standard_normal((n, n))] * T
            if j < N - 1 and i != 2:
                kw["east"] = [0.1 * rng.standard_normal((n, n))] * T
            row.append(SubsystemData(n=n, m=m, A=[a] * T, B=[rng.standard_normal((n, m))] * T,
                                     Q=[np.eye(n)] * (T + 1), R=[np.eye(m)] * T, **kw))
            irow.append(rng.standard_normal(n))
        subs.append(row)
        init.append(irow)
    return GridLQProblem(K, N, T, subs, BoundaryData(init=init))


def hetero_problem(K=3, N=4, T=4, seed=21):
    """Mixed state (1..3) and input (1..2) dimensions (grid_problem.py:103-141): couplings
    map the neighbour's state into the node's, every block stage-invariant, a boundary
    trajectory on the north edge."""
    rng = np.random.default_rng(seed)
    nd = [[1 + (i + 2 * j) % 3 for j in range(N)] for i in range(K)]
    md = [[1 + (i + j) % 2 for j in range(N)] for i in range(K)]
    nbr = {"west": (0, -1), "east": (0, 1), "north": (-1, 0), "south": (1, 0)}
    subs, init = [], []
    for i in range(K):
        row, irow = [], []
        for j in range(N):
            n, m = nd[i][j], md[i][j]
            a = 0.6 * np.eye(n) + 0.15 * rng.uniform(-1, 1, (n, n))
            q = np.eye(n) * rng.uniform(1.0, 3.0) + 0.1 * np.ones((n, n))
            r = np.eye(m) * rng.uniform(0.5, 2.0)
            kw = {}
            for d, (di, dj) in nbr.items():
                ii, jj = i + di, j + dj
                inside = 0 <= ii < K and 0 <= jj < N
                if not inside and d != "north":
                    continue                            # only the north edge has a trajectory
                cols = nd[ii][jj] if inside else n      # off-grid: boundary signal of size n
                kw[d] = [0.08 * rng.uniform(-1, 1, (n, cols))] * T
            row.append(SubsystemData(n=n, m=m, A=[a] * T, B=[rng.uniform(-1, 1, (n, m))] * T,
                                     Q=[q] * (T + 1), R=[r] * T, **kw))
            irow.append(rng.uniform(-1, 1, n))
        subs.append(row)
        init.append(irow)
    north = [[rng.uniform(-1, 1, nd[0][j]) for _ in range(T)] for j in range(N)]
    return GridLQProblem(K, N, T, subs, BoundaryData(init=init, north=north))
