"""The reference's deterministic multiply counters, reproduced from block structure.

``SolveReport.op_counts`` (``pcg.py:19-28,76-131``) accumulates scalar-multiply counts
derived from which blocks the reference *stores*, not from their values.  This module
recomputes those counts from ``GridArrays`` so the B200 path reports identical numbers:

* ``matvec_flops``         -- SchurOperator.matvec_flops (``kkt_assembly.py:429-437``)
* ``outer_coupling_flops`` -- ``kkt_assembly.py:439-444``
* ``inner_coupling_flops`` -- PairSplitting.inner_coupling_flops (``kkt_assembly.py:664-675``)
* ``pair_solve_flops``     -- sum of BlockTridiagCholesky.solve_flops (``block_linalg.py:326-330``)
* ``apply_flops``          -- NestedJacobiPreconditioner.apply_flops (``nested_jacobi.py:53-61``)

Block-existence rules (``kkt_assembly.py:215-254``): the within-column piece of Ahat
stores A at (i,i), north at (i,i-1) when declared and i>0, south at (i,i+1) when
declared and i<K-1; the west/east column pieces exist only if some coupling in that
column is nonzero, and then store all K diagonal blocks.  Xi_t mirrors Ahat_t's blocks;
Psi_t stores (a,b) whenever some node s has stored Ahat blocks (a,s) and (b,s)
(``_accumulate_product``, ``kkt_assembly.py:310-323``), plus every diagonal block.
"""

from __future__ import annotations

import numpy as np

from .problem import GridArrays

OFF13 = ((0, 0), (-1, 0), (1, 0), (0, -1), (0, 1), (-2, 0), (2, 0), (0, -2), (0, 2),
         (-1, -1), (-1, 1), (1, -1), (1, 1))
OFF5 = OFF13[:5]


def _shift(mask, di, dj):
    """out[j, i] = mask[j+dj, i+di] (False outside)."""
    N, K = mask.shape
    out = np.zeros_like(mask)
    out[max(0, -dj):min(N, N - dj), max(0, -di):min(K, K - di)] = \
        mask[max(0, dj):min(N, N + dj), max(0, di):min(K, K + di)]
    return out


def ahat_exists(ga: GridArrays, dc: int):
    """[5, N, K] bool: Ahat(a, a+OFF5[u]) is a stored block for dynamics set dc."""
    K, N = ga.K, ga.N
    ii = np.arange(K)[None, :]
    jj = np.arange(N)[:, None]
    out = np.zeros((5, N, K), dtype=bool)
    out[0] = True
    out[1] = (ii > 0) & ga.cmask[2]
    out[2] = (ii < K - 1) & ga.cmask[3]
    west_piece = np.any(ga.C[dc, 0] != 0, axis=(1, 2, 3))   # per column j
    east_piece = np.any(ga.C[dc, 1] != 0, axis=(1, 2, 3))
    out[3] = (jj > 0) & west_piece[:, None]
    out[4] = (jj < N - 1) & east_piece[:, None]
    return out


def psi_exists(ga: GridArrays, dc: int):
    """[13, N, K] bool: Psi_t(a, a+OFF13[o]) stored, for stages t>=1 using dynamics dc."""
    ex = ahat_exists(ga, dc)
    out = np.zeros((13, ga.N, ga.K), dtype=bool)
    out[0] = True
    for o in range(1, 13):
        di, dj = OFF13[o]
        acc = np.zeros((ga.N, ga.K), dtype=bool)
        for u in range(5):
            for w in range(5):
                if OFF5[u][0] - OFF5[w][0] == di and OFF5[u][1] - OFF5[w][1] == dj:
                    acc |= ex[u] & _shift(ex[w], di, dj)
        out[o] = acc & _shift(np.ones((ga.N, ga.K), dtype=bool), di, dj)
    return out


def _cross_pair(N, dj):
    jj = np.arange(N)
    return (jj + dj) // 2 != jj // 2


def counters(ga: GridArrays, inner_sweeps: int, outer_sweeps: int, nd=None) -> dict:
    """``nd`` [N][K]: the true state dimensions when ``ga`` is the padded embedding of a
    problem with mixed dimensions (embed.py); a stored block (a, b) then costs n_a n_b."""
    n = ga.n
    T = ga.T
    dims = np.full((ga.N, ga.K), n, dtype=np.int64) if nd is None else np.asarray(nd, dtype=np.int64)

    def weight(mask, off):
        """sum over stored blocks (a, a+off) of n_a * n_{a+off}"""
        di, dj = off
        return int(np.sum(mask * dims * _shift(dims, di, dj)))

    per_dc = {}
    for dc in np.unique(ga.dyn_class):
        ex = ahat_exists(ga, int(dc))
        # only in-grid targets count (off-grid existence flags are already False)
        ps = psi_exists(ga, int(dc))
        cross = 0
        for o in range(1, 13):
            dj = OFF13[o][1]
            if dj == 0:
                continue
            cross += weight(ps[o] & _cross_pair(ga.N, dj)[:, None], OFF13[o])
        per_dc[int(dc)] = dict(ahat=sum(weight(ex[u], OFF5[u]) for u in range(5)),
                               psi=sum(weight(ps[o], OFF13[o]) for o in range(13)),
                               cross=cross)
    matvec = int(np.sum(dims * dims))        # Psi_0 = Qinv_0: diagonal blocks only
    outer = 0
    inner = 0
    for t in range(T):
        st = per_dc[int(ga.dyn_class[t])]
        matvec += st["psi"] + 2 * st["ahat"]               # Psi_{t+1} and Xi_t (both ways)
        outer += 2 * st["ahat"]
        inner += st["cross"]
    # pair solves: every (v, t) chain, block k holds the states of rows 2k, 2k+1 of the pair
    pair = 0
    for v in range((ga.N + 1) // 2):
        prev = None
        for k in range((ga.K + 1) // 2):
            q = int(dims[2 * v:2 * v + 2, 2 * k:2 * k + 2].sum())
            pair += 2 * q * q + (2 * q * prev if prev is not None else 0)
            prev = q
    pair *= T + 1
    l, s = int(inner_sweeps), int(outer_sweeps)
    apply = s * l * pair + s * (l - 1) * inner + (s - 1) * outer
    return {
        "matvec_flops": matvec,
        "outer_coupling_flops": outer,
        "inner_coupling_flops": inner,
        "pair_solve_flops": pair,
        "apply_flops": apply,
    }
