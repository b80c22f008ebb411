"""Seeded synthetic problems for the BASELINE.json configurations.

The reference ships no generator for these configs (SURVEY.md finding 3), so they are
defined here, emitting ``GridArrays`` directly (and a byte-identical ``GridLQProblem``
view via ``problem.arrays_to_problem`` for the oracle / reference).  Draw order is
fixed and documented per generator so the same seed always gives the same bytes.

* ``random_case``  -- configs 1, 3, 5: A = G * rho / rho(G) with G ~ N(0,1) per node;
  couplings to every in-grid 4-neighbour ~ N(0, std^2); B ~ N(0,1); Q = I or
  diag(U[1,10]); R = I; x0 ~ N(0,1); terminal weight Q_T = Q.
* ``msd_case``     -- configs 2, 4: 2-D mass-spring-damper grid, n=2 (position,
  velocity), m=1; masses U[0.8,1.2] per node, spring k ~ U[0.5,1.5] and damper
  c ~ U[0.1,0.5] per in-grid edge (no walls); forward Euler with dt=0.1;
  Q = diag(10,1), R = 0.1; x0 = (U[-1,1], 0).
"""

from __future__ import annotations

import numpy as np

from .problem import GridArrays

EULER_STEP = 0.1

# direction order (west, east, north, south) and the (di, dj) of each neighbour
_DIRS = ((0, -1), (0, 1), (-1, 0), (1, 0))


def _in_grid_mask(K, N):
    """cmask[d, j, i]: neighbour in direction d exists."""
    j = np.arange(N)[:, None]
    i = np.arange(K)[None, :]
    out = np.zeros((4, N, K), dtype=bool)
    for d, (di, dj) in enumerate(_DIRS):
        out[d] = (i + di >= 0) & (i + di < K) & (j + dj >= 0) & (j + dj < N)
    return out


def _offset_from_init(K, N, T, n, x0):
    """omega~ for problems without boundary trajectories: x0 at stage 0, zeros after
    (``kkt_assembly.py:275-279``).  x0 has shape [N, K, n]."""
    off = np.zeros(K * N * n * (T + 1))
    off[: K * N * n] = x0.reshape(-1)
    return off


def random_case(K, N, T, n, m, seed, rho=0.9, coupling_std=0.05, q_diag_range=None):
    """Random stable subsystems (BASELINE configs 1, 3, 5).

    Draw order from ``np.random.default_rng(seed)``: G [N,K,n,n]; couplings [4,N,K,n,n];
    B [N,K,n,m]; Q diagonals [N,K,n] (only when ``q_diag_range`` is given); x0 [N,K,n].
    """
    rng = np.random.default_rng(seed)
    g = rng.standard_normal((N, K, n, n))
    radius = np.max(np.abs(np.linalg.eigvals(g)), axis=-1)
    a = g * (rho / radius)[..., None, None]
    cmask = _in_grid_mask(K, N)
    c = rng.standard_normal((4, N, K, n, n)) * coupling_std
    c = c * cmask[..., None, None]
    b = rng.standard_normal((N, K, n, m))
    if q_diag_range is None:
        q = np.broadcast_to(np.eye(n), (N, K, n, n)).copy()
    else:
        lo, hi = q_diag_range
        diag = rng.uniform(lo, hi, size=(N, K, n))
        q = np.zeros((N, K, n, n))
        idx = np.arange(n)
        q[..., idx, idx] = diag
    r = np.broadcast_to(np.eye(m), (N, K, m, m)).copy()
    x0 = rng.standard_normal((N, K, n))
    return GridArrays(
        K=K, N=N, T=T, n=n, m=m,
        A=a[None], B=b[None], R=r[None], C=c[None], cmask=cmask, Q=q[None],
        dyn_class=np.zeros(T, dtype=np.int32), cost_class=np.zeros(T + 1, dtype=np.int32),
        offset=_offset_from_init(K, N, T, n, x0),
    )


def msd_case(K, N, T, seed):
    """2-D mass-spring-damper grid (BASELINE configs 2 and 4).

    Draw order: masses [N,K]; horizontal-edge springs [N-1,K] and dampers [N-1,K]
    (edge between columns j and j+1); vertical-edge springs [N,K-1] and dampers [N,K-1]
    (edge between rows i and i+1); initial positions [N,K].
    """
    rng = np.random.default_rng(seed)
    h = EULER_STEP
    mass = rng.uniform(0.8, 1.2, size=(N, K))
    kh = rng.uniform(0.5, 1.5, size=(max(N - 1, 0), K))
    ch = rng.uniform(0.1, 0.5, size=(max(N - 1, 0), K))
    kv = rng.uniform(0.5, 1.5, size=(N, max(K - 1, 0)))
    cv = rng.uniform(0.1, 0.5, size=(N, max(K - 1, 0)))
    pos = rng.uniform(-1.0, 1.0, size=(N, K))

    # per node and direction: the edge parameters toward that neighbour (0 off-grid)
    ke = np.zeros((4, N, K))
    ce = np.zeros((4, N, K))
    ke[0, 1:, :], ce[0, 1:, :] = kh, ch          # west edge of column j>0
    ke[1, :-1, :], ce[1, :-1, :] = kh, ch        # east edge of column j<N-1
    ke[2, :, 1:], ce[2, :, 1:] = kv, cv          # north edge of row i>0
    ke[3, :, :-1], ce[3, :, :-1] = kv, cv        # south edge of row i<K-1
    ksum = ke.sum(axis=0)
    csum = ce.sum(axis=0)

    a = np.zeros((N, K, 2, 2))
    a[..., 0, 0] = 1.0
    a[..., 0, 1] = h
    a[..., 1, 0] = -h * ksum / mass
    a[..., 1, 1] = 1.0 - h * csum / mass
    cmask = _in_grid_mask(K, N)
    c = np.zeros((4, N, K, 2, 2))
    c[..., 1, 0] = h * ke / mass
    c[..., 1, 1] = h * ce / mass
    c = c * cmask[..., None, None]
    b = np.zeros((N, K, 2, 1))
    b[..., 1, 0] = h / mass
    q = np.broadcast_to(np.diag([10.0, 1.0]), (N, K, 2, 2)).copy()
    r = np.full((N, K, 1, 1), 0.1)
    x0 = np.stack([pos, np.zeros_like(pos)], axis=-1)
    return GridArrays(
        K=K, N=N, T=T, n=2, m=1,
        A=a[None], B=b[None], R=r[None], C=c[None], cmask=cmask, Q=q[None],
        dyn_class=np.zeros(T, dtype=np.int32), cost_class=np.zeros(T + 1, dtype=np.int32),
        offset=_offset_from_init(K, N, T, 2, x0),
    )


# BASELINE.json configurations ------------------------------------------------------------

def config1(seed=0):
    """Tiny CPU-runnable case: 4x4, T=20, n=2, m=1, rho 0.9, coupling std 0.05."""
    return random_case(4, 4, 20, 2, 1, seed, rho=0.9, coupling_std=0.05)


def config2(seed=0, K=16, N=16, T=50):
    """Mass-spring-damper 16x16, T=50."""
    return msd_case(K, N, T, seed)


def config3(seed=0, K=64, N=64, T=100):
    """Random 64x64, T=100, n=4, m=2, rho 0.95, coupling std 0.02, Q = diag(U[1,10])."""
    return random_case(K, N, T, 4, 2, seed, rho=0.95, coupling_std=0.02, q_diag_range=(1.0, 10.0))


def config4(seed=0, K=256, N=256, T=200):
    """Headline: mass-spring-damper 256x256, T=200."""
    return msd_case(K, N, T, seed)


def config5(seed=0, K=32, N=1024, T=500):
    """Block-size / aspect stress: 32x1024, T=500, n=8, m=4, rho 0.9, coupling std 0.01."""
    return random_case(K, N, T, 8, 4, seed, rho=0.9, coupling_std=0.01, q_diag_range=(1.0, 10.0))


CONFIGS = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}
