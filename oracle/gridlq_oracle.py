"""CPU oracle for the gridlq PCGM hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference algorithm (``gridlq`` v0.1.0 under
/root/reference/pkg/src/gridlq).  It exists to check the B200 path: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / ``--impl reference`` leg
may import it.  The product (``paper_2304_04980_b200``) never imports or calls it and
has no CPU fallback.

Pinned: ``tests/test_oracle_golden.py`` checks every function here against golden
vectors produced by running the reference itself (``oracle/make_golden.py`` ->
``tests/golden/*.npz``).

What is restated (file:line in the reference):

* ``spd_inverse``        -- block_linalg.py:43-85 (column Cholesky, pivot rule
  PIVOT_RTOL * max diag, forward-substitution inverse, Linv' Linv symmetrised)
* ``Oracle.psi``         -- stage diagonals Psi_t of build_schur, kkt_assembly.py:487-533
* ``Oracle.xi``          -- stage couplings Xi_t = -Ahat_t Qinv_t, kkt_assembly.py:535-543
* ``Oracle.apply_delta`` -- SchurOperator.apply, kkt_assembly.py:379-403
* ``Oracle.apply_outer`` -- SchurOperator.apply_outer_coupling, kkt_assembly.py:414-425
* ``Oracle.apply_inner`` -- PairSplitting.apply_inner_coupling, kkt_assembly.py:645-662
* ``Oracle.factors``     -- PairSplitting._extract + pair_rows + block_tridiag_factor,
  kkt_assembly.py:605-641, block_linalg.py:277-301, 371-398
* ``Oracle.pair_solve``  -- BlockTridiagCholesky.solve, block_linalg.py:336-358
* ``Oracle.apply_precond`` -- NestedJacobiPreconditioner.apply / inner_sweep,
  nested_jacobi.py:79-122
* ``pcg``                -- pcg_solve, pcg.py:50-149

Vectors use the reference order (t, j, i, k) and are reshaped to [T+1, N, K, n] here.
Grid neighbours missing at an edge contribute zero blocks.  Odd K / odd N (ragged last
row block / singleton last column pair) are handled by padding the pair chains with
identity rows, which leaves the real rows' factors unchanged.
"""

from __future__ import annotations

import math

import numpy as np

PIVOT_RTOL = 1e-14

# 13-point diamond (di, dj); the first five form the 5-point stencil
OFF13 = ((0, 0), (-1, 0), (1, 0), (0, -1), (0, 1), (-2, 0), (2, 0), (0, -2), (0, 2),
         (-1, -1), (-1, 1), (1, -1), (1, 1))
OFF5 = OFF13[:5]
# 5-point slot -> coupling direction index (west, east, north, south) of the owner
_DIR_OF_SLOT = {1: 2, 2: 3, 3: 0, 4: 1}
# slot of the opposite offset
_OPP5 = {0: 0, 1: 2, 2: 1, 3: 4, 4: 3}


class OracleError(Exception):
    pass


class NotSPD(OracleError):
    pass


# ---------------------------------------------------------------------------
# dense kernels (block_linalg.py:43-85), batched over leading axes


def cholesky(m, real_mask=None):
    """Unblocked column Cholesky (block_linalg.py:43-65), batched.

    ``real_mask`` marks real (non-padding) positions: the pivot threshold uses the max
    diagonal over real positions only, so padding never changes the decision."""
    m = np.asarray(m, dtype=float)
    n = m.shape[-1]
    lower = np.zeros_like(m)
    diag = np.diagonal(m, axis1=-2, axis2=-1)
    if real_mask is not None:
        diag = np.where(real_mask, diag, -np.inf)
    tol = PIVOT_RTOL * np.max(diag, axis=-1)
    for j in range(n):
        piv = m[..., j, j] - np.einsum("...k,...k->...", lower[..., j, :j], lower[..., j, :j])
        if np.any(piv <= tol):
            bad = np.argwhere(piv <= tol)[0]
            raise NotSPD(f"pivot {piv[tuple(bad)]:.3e} at index {j} (threshold {tol[tuple(bad)]:.3e})")
        ljj = np.sqrt(piv)
        lower[..., j, j] = ljj
        if j + 1 < n:
            lower[..., j + 1:, j] = (
                m[..., j + 1:, j]
                - np.einsum("...rk,...k->...r", lower[..., j + 1:, :j], lower[..., j, :j])
            ) / ljj[..., None]
    return lower


def lower_inverse(lower):
    """Forward-substitution inverse (block_linalg.py:68-78), batched."""
    n = lower.shape[-1]
    inv = np.zeros_like(lower)
    for i in range(n):
        row = -np.einsum("...k,...kc->...c", lower[..., i, :i], inv[..., :i, :])
        row[..., i] += 1.0
        inv[..., i, :] = row / lower[..., i, i][..., None]
    return inv


def spd_inverse(m):
    """block_linalg.py:81-85."""
    linv = lower_inverse(cholesky(m))
    inv = np.swapaxes(linv, -1, -2) @ linv
    return 0.5 * (inv + np.swapaxes(inv, -1, -2))


def mv(mat, vec):
    """Batched small matvec: out[..., a] = sum_b mat[..., a, b] * vec[..., b] (b ascending)."""
    out = mat[..., :, 0] * vec[..., None, 0]
    for b in range(1, mat.shape[-1]):
        out = out + mat[..., :, b] * vec[..., None, b]
    return out


def shift(x, di, dj):
    """s[..., j, i, :] = x[..., j+dj, i+di, :] (zero outside the grid); axes [..., N, K, n]."""
    N, K = x.shape[-3], x.shape[-2]
    out = np.zeros_like(x)
    js = slice(max(0, -dj), min(N, N - dj))
    is_ = slice(max(0, -di), min(K, K - di))
    jd = slice(max(0, dj), min(N, N + dj))
    id_ = slice(max(0, di), min(K, K + di))
    out[..., js, is_, :] = x[..., jd, id_, :]
    return out


def shift_blocks(b, di, dj):
    """Same as ``shift`` for per-node blocks with axes [N, K, r, c]."""
    N, K = b.shape[0], b.shape[1]
    out = np.zeros_like(b)
    js = slice(max(0, -dj), min(N, N - dj))
    is_ = slice(max(0, -di), min(K, K - di))
    jd = slice(max(0, dj), min(N, N + dj))
    id_ = slice(max(0, di), min(K, K + di))
    out[js, is_] = b[jd, id_]
    return out


def _before(di, dj):
    """Neighbour at (di, dj) precedes the node in the (j, i) global order."""
    return dj < 0 or (dj == 0 and di < 0)


class Oracle:
    """Operators of one problem (GridArrays-shaped input: attributes K, N, T, n, m, A, B,
    R, C, Q, dyn_class, cost_class, offset)."""

    def __init__(self, ga, inner_sweeps=2, outer_sweeps=2):
        if inner_sweeps < 1 or outer_sweeps < 1:
            raise ValueError("sweep budgets must be at least 1")  # nested_jacobi.py:33-34
        self.K, self.N, self.T, self.n, self.m = ga.K, ga.N, ga.T, ga.n, ga.m
        self.L, self.S = int(inner_sweeps), int(outer_sweeps)
        self.T1 = self.T + 1
        self.dim = self.K * self.N * self.n * self.T1
        self.offset = np.asarray(ga.offset, dtype=float)
        dyn = np.asarray(ga.dyn_class)
        cost = np.asarray(ga.cost_class)
        # kkt_assembly.py:256-273 -- Q^-1 and R^-1 through spd_inverse
        self.qinv = spd_inverse(ga.Q)
        rinv = spd_inverse(ga.R)
        brb = (ga.B @ rinv) @ np.swapaxes(ga.B, -1, -2)
        self.brb = 0.5 * (brb + np.swapaxes(brb, -1, -2))        # kkt_assembly.py:525-526
        # Ahat 5-point blocks per dynamics set: [nd, N, K, 5, n, n] = A, north, south, west, east
        self.ahat = np.stack([ga.A, ga.C[:, 2], ga.C[:, 3], ga.C[:, 0], ga.C[:, 1]], axis=3)
        # stage classes
        self.psi_key, self.psi_cls = [], np.empty(self.T1, dtype=int)
        for t in range(self.T1):
            key = (int(cost[0]), -1, -1) if t == 0 else (int(cost[t]), int(dyn[t - 1]), int(cost[t - 1]))
            if key not in self.psi_key:
                self.psi_key.append(key)
            self.psi_cls[t] = self.psi_key.index(key)
        self.xi_key, self.xi_cls = [], np.empty(self.T, dtype=int)
        for t in range(self.T):
            key = (int(dyn[t]), int(cost[t]))
            if key not in self.xi_key:
                self.xi_key.append(key)
            self.xi_cls[t] = self.xi_key.index(key)
        self.psi = [self._assemble_psi(*k) for k in self.psi_key]
        self.xi, self.xit = zip(*[self._assemble_xi(*k) for k in self.xi_key]) if self.T else ((), ())
        self.V = (self.N + 1) // 2
        self.nb = (self.K + 1) // 2
        self.q = 4 * self.n
        self.factors = [self._factor(p) for p in self.psi]

    # -- assembly ------------------------------------------------------------------

    def _assemble_xi(self, dc, qc):
        """Xi(a, a+u) = -Ahat(a, a+u) Qinv(a+u); XiT(a, u) = Xi(a+u, a)' (kkt_assembly.py:535-543)."""
        ah = self.ahat[dc]
        qi = self.qinv[qc]
        xi = np.zeros_like(ah)
        xit = np.zeros_like(ah)
        for u, (di, dj) in enumerate(OFF5):
            q_at = shift_blocks(qi, di, dj)
            xi[:, :, u] = -(ah[:, :, u] @ q_at)
            # Xi(p, a) with p = a+u: owner p's block toward a is its opposite slot
            owner = shift_blocks(ah[:, :, _OPP5[u]], di, dj)
            xit[:, :, u] = np.swapaxes(-(owner @ qi), -1, -2)
        return xi, xit

    def _assemble_psi(self, qc, dc, qp):
        """13 blocks Psi(a, a+off13[o]) per node (kkt_assembly.py:493-533)."""
        n = self.n
        psi = np.zeros((self.N, self.K, 13, n, n))
        psi[:, :, 0] = self.qinv[qc]
        if dc < 0:
            return psi
        ah = self.ahat[dc]
        qprev = self.qinv[qp]
        # pre[u] = Ahat(a, a+u) Qinv(a+u)
        pre = np.stack([ah[:, :, u] @ shift_blocks(qprev, *OFF5[u]) for u in range(5)], axis=2)
        # order of the common nodes s by global order (j, then i)
        order5 = sorted(range(5), key=lambda u: (OFF5[u][1], OFF5[u][0]))
        diag = psi[:, :, 0].copy()
        for u in order5:
            diag = diag + pre[:, :, u] @ np.swapaxes(ah[:, :, u], -1, -2)
        diag = diag + self.brb[dc]
        psi[:, :, 0] = 0.5 * (diag + np.swapaxes(diag, -1, -2))
        for o in range(1, 13):
            di, dj = OFF13[o]
            pairs = [(u, w) for u in range(5) for w in range(5)
                     if OFF5[u][0] - OFF5[w][0] == di and OFF5[u][1] - OFF5[w][1] == dj]
            # common nodes s = a+u sorted by global order
            pairs.sort(key=lambda uw: (OFF5[uw[0]][1], OFF5[uw[0]][0]))
            if _before(di, dj):
                acc = np.zeros((self.N, self.K, n, n))
                for u, w in pairs:
                    acc = acc + pre[:, :, u] @ np.swapaxes(shift_blocks(ah[:, :, w], di, dj), -1, -2)
                blk = acc
            else:
                # canonical owner is b = a+o: compute Psi(b, a) there and transpose
                acc = np.zeros((self.N, self.K, n, n))
                for u, w in pairs:
                    acc = acc + shift_blocks(pre[:, :, w], di, dj) @ np.swapaxes(ah[:, :, u], -1, -2)
                blk = np.swapaxes(acc, -1, -2)
            # zero outside the grid
            mask = np.zeros((self.N, self.K), dtype=bool)
            mask[max(0, -dj):min(self.N, self.N - dj), max(0, -di):min(self.K, self.K - di)] = True
            psi[:, :, o] = blk * mask[:, :, None, None]
        return psi

    # -- pair splitting and factorisation ------------------------------------------

    def _local_pos(self):
        """(ri, ci, kk) of every pair-local position p = (ri*2 + ci)*n + kk."""
        out = []
        for ri in range(2):
            for ci in range(2):
                for kk in range(self.n):
                    out.append((ri, ci, kk))
        return out

    def _pair_blocks(self, psi, k, prev):
        """M_kk (prev=False) or M_{k,k-1} (prev=True), batched over pairs v: [V, q, q]."""
        n, q, V = self.n, self.q, self.V
        pos = self._local_pos()
        out = np.zeros((V, q, q))
        vs = np.arange(V)
        for p, (ri, ci, kk) in enumerate(pos):
            i = 2 * k + ri
            if i >= self.K:
                continue
            j = 2 * vs + ci
            for p2, (ri2, ci2, kk2) in enumerate(pos):
                i2 = 2 * (k - 1) + ri2 if prev else 2 * k + ri2
                di, dj = i2 - i, ci2 - ci
                if abs(di) + abs(dj) > 2 or i2 < 0 or i2 >= self.K:
                    continue
                o = OFF13.index((di, dj))
                ok = (j < self.N) & (j + dj < self.N)
                out[ok, p, p2] = psi[j[ok], i, o, kk, kk2]
        return out

    def _real(self, k):
        """[V, q] mask of real positions in block k."""
        mask = np.zeros((self.V, self.q), dtype=bool)
        for p, (ri, ci, kk) in enumerate(self._local_pos()):
            for v in range(self.V):
                mask[v, p] = (2 * k + ri < self.K) and (2 * v + ci < self.N)
        return mask

    def _factor(self, psi):
        """block_tridiag_factor on every pair chain (block_linalg.py:371-398)."""
        V, q = self.V, self.q
        linv = np.zeros((self.nb, V, q, q))
        sub = np.zeros((self.nb, V, q, q))
        for k in range(self.nb):
            mkk = self._pair_blocks(psi, k, prev=False)
            real = self._real(k)
            # padding: identity on padded diagonal positions
            idx = np.arange(q)
            mkk[:, idx, idx] = np.where(real, mkk[:, idx, idx], 1.0)
            if k:
                mk = self._pair_blocks(psi, k, prev=True)
                coupling = mk @ np.swapaxes(linv[k - 1], -1, -2)
                schur = mkk - coupling @ np.swapaxes(coupling, -1, -2)
                schur = 0.5 * (schur + np.swapaxes(schur, -1, -2))
                sub[k] = coupling
            else:
                schur = mkk
            lo = cholesky(schur, real_mask=real)
            linv[k] = lower_inverse(lo)
        return linv, sub

    # -- vector layout helpers --------------------------------------------------------

    def as_grid(self, x):
        return np.asarray(x, dtype=float).reshape(self.T1, self.N, self.K, self.n)

    def to_local(self, xg, ts):
        """[nt, N, K, n] -> [V, nb, q, nt] pair-local interleaved order."""
        nt = len(ts)
        xp = np.zeros((nt, 2 * self.V, 2 * self.nb, self.n))
        xp[:, : self.N, : self.K] = xg
        xp = xp.reshape(nt, self.V, 2, self.nb, 2, self.n)       # t, v, ci, k, ri, kk
        return np.ascontiguousarray(xp.transpose(1, 3, 4, 2, 5, 0)).reshape(
            self.V, self.nb, self.q, nt)

    def from_local(self, loc, nt):
        xp = loc.reshape(self.V, self.nb, 2, 2, self.n, nt).transpose(5, 0, 3, 1, 2, 4)
        xp = xp.reshape(nt, 2 * self.V, 2 * self.nb, self.n)
        return xp[:, : self.N, : self.K]

    # -- operators ----------------------------------------------------------------------

    def _class_stages(self, cls):
        groups = {}
        for t, c in enumerate(cls):
            groups.setdefault(int(c), []).append(t)
        return groups

    def apply_delta(self, x):
        """SchurOperator.apply (kkt_assembly.py:379-403)."""
        xg = self.as_grid(x)
        y = np.zeros_like(xg)
        for c, ts in self._class_stages(self.psi_cls).items():
            for o, (di, dj) in enumerate(OFF13):
                y[ts] += mv(self.psi[c][None, :, :, o], shift(xg[ts], di, dj))
        for c, ts in self._class_stages(self.xi_cls).items():
            ts = np.array(ts)
            for u, (di, dj) in enumerate(OFF5):
                # Xi_t x_t into row t+1 ; Xi_t' x_{t+1} into row t
                y[ts + 1] += mv(self.xi[c][None, :, :, u], shift(xg[ts], di, dj))
                y[ts] += mv(self.xit[c][None, :, :, u], shift(xg[ts + 1], di, dj))
        return y.reshape(-1)

    def apply_outer(self, x):
        """SchurOperator.apply_outer_coupling (kkt_assembly.py:414-425)."""
        xg = self.as_grid(x)
        y = np.zeros_like(xg)
        for c, ts in self._class_stages(self.xi_cls).items():
            ts = np.array(ts)
            for u, (di, dj) in enumerate(OFF5):
                y[ts + 1] -= mv(self.xi[c][None, :, :, u], shift(xg[ts], di, dj))
                y[ts] -= mv(self.xit[c][None, :, :, u], shift(xg[ts + 1], di, dj))
        return y.reshape(-1)

    def apply_inner(self, x):
        """PairSplitting.apply_inner_coupling (kkt_assembly.py:645-662): minus the
        cross-pair blocks of the stage diagonals."""
        xg = self.as_grid(x)
        y = np.zeros_like(xg)
        jj = np.arange(self.N)
        for c, ts in self._class_stages(self.psi_cls).items():
            for o, (di, dj) in enumerate(OFF13):
                if dj == 0:
                    continue
                cross = ((jj + dj) // 2 != jj // 2)[:, None, None, None]
                blk = self.psi[c][:, :, o] * cross
                y[ts] -= mv(blk[None], shift(xg[ts], di, dj))
        return y.reshape(-1)

    def pair_solve(self, rhs):
        """Phi~^-1 rhs: every (pair, stage) chain (nested_jacobi.py:65-77 ->
        block_linalg.py:336-358)."""
        xg = self.as_grid(rhs)
        out = np.zeros_like(xg)
        for c, ts in self._class_stages(self.psi_cls).items():
            linv, sub = self.factors[c]
            b = self.to_local(xg[ts], ts)                 # [V, nb, q, nt]
            work = np.empty_like(b)
            for k in range(self.nb):
                seg = b[:, k]
                if k:
                    seg = seg - sub[k] @ work[:, k - 1]
                work[:, k] = linv[k] @ seg
            for k in range(self.nb - 1, -1, -1):
                seg = work[:, k]
                if k + 1 < self.nb:
                    seg = seg - np.swapaxes(sub[k + 1], -1, -2) @ work[:, k + 1]
                work[:, k] = np.swapaxes(linv[k], -1, -2) @ seg
            out[ts] = self.from_local(work, len(ts))
        return out.reshape(-1)

    def inner_sweep(self, rhs, start=None):
        """nested_jacobi.py:79-103: L sweeps from the zero start, or L sweeps warm-started
        from `start` (the standalone iteration)."""
        if start is None:
            theta = self.pair_solve(rhs)
            remaining = self.L - 1
        else:
            theta = start
            remaining = self.L
        for _ in range(remaining):
            theta = self.pair_solve(rhs + self.apply_inner(theta))
        return theta

    def nbjm_solve(self, rhs, tol=1e-9, max_outer=50000):
        """NestedJacobiPreconditioner.solve (nested_jacobi.py:124-151).  Returns
        (solution, outer sweeps, converged); on budget exhaustion the solution is the last
        iterate (the reference raises MaxIterationsExceeded carrying it)."""
        rhs = np.asarray(rhs, dtype=float)
        delta = None
        for s in range(max_outer):
            if delta is None:
                new = self.inner_sweep(rhs)
                prev = np.zeros_like(new)
            else:
                new = self.inner_sweep(rhs + self.apply_outer(delta), start=delta)
                prev = delta
            if float(np.max(np.abs(new - prev))) < tol:
                return new, s + 1, True
            delta = new
        return delta, max_outer, False

    def apply_precond(self, r):
        """NestedJacobiPreconditioner.apply (nested_jacobi.py:105-122)."""
        if self.L % 2:
            raise ValueError("preconditioner use requires an even inner budget "
                             f"(got {self.L}); odd budgets are standalone-only")
        r = np.asarray(r, dtype=float)
        delta = self.inner_sweep(r)
        for _ in range(self.S - 1):
            delta = self.inner_sweep(r + self.apply_outer(delta))
        return delta


def pcg(oracle, rhs, tol=1e-9, max_steps=None, x0=None, precond=True, callback=None):
    """pcg_solve's control flow (pcg.py:50-149).

    Returns (x, history, steps, converged, status) where status is "ok", "max_steps" or
    "breakdown" (the reference raises MaxIterationsExceeded / BreakdownError there)."""
    rhs = np.asarray(rhs, dtype=float)
    n = oracle.dim
    if max_steps is None:
        max_steps = n + 50
    if x0 is None:
        x = np.zeros(n)
        r = rhs.copy()
    else:
        x = np.array(x0, dtype=float, copy=True)
        r = rhs - oracle.apply_delta(x)
    d = oracle.apply_precond(r) if precond else r.copy()
    mu = float(d @ r)
    history = []
    converged = False
    steps = 0
    for _ in range(max_steps):
        y = oracle.apply_delta(d)
        curvature = float(y @ d)
        if curvature <= 0.0:
            return x, history, steps, False, "breakdown"
        alpha = mu / curvature
        x += alpha * d
        r = r - alpha * y
        res = float(np.max(np.abs(r)))
        history.append(res)
        steps += 1
        if callback is not None:
            callback(steps, x, r)
        if res < tol:
            converged = True
            break
        q = oracle.apply_precond(r) if precond else r
        mu_next = float(q @ r)
        d = q + (mu_next / mu) * d
        mu = mu_next
    return x, history, steps, converged, ("ok" if converged else "max_steps")


def step_cost_model(dim, S, L):
    """SURVEY.md 8(d) canonical bytes per PCGM step: 8*dim*C(S,L)."""
    return 8 * dim * (10 + (3 * L - 1) + (S - 1) * (4 * L - 1))


__all__ = ["Oracle", "pcg", "spd_inverse", "cholesky", "lower_inverse", "NotSPD",
           "OFF13", "OFF5", "step_cost_model", "math"]


# ---- primal recovery and KKT residuals (recovery.py:50-80, kkt_assembly.py:84-160) ------------
# TEST INFRASTRUCTURE ONLY, like everything in oracle/.

_DIRS = ((0, -1), (0, 1), (-1, 0), (1, 0))   # C direction order (west, east, north, south)


def _shift(X, di, dj):
    """Z[j, i] = X[j + dj, i + di] (zero outside the grid); X is [N, K, ...]."""
    Z = np.zeros_like(X)
    N, K = X.shape[:2]
    js = slice(max(0, -dj), min(N, N - dj))
    jd = slice(max(0, dj), min(N, N + dj))
    is_ = slice(max(0, -di), min(K, K - di))
    id_ = slice(max(0, di), min(K, K + di))
    Z[js, is_] = X[jd, id_]
    return Z


def _unshift(Y, di, dj):
    """adjoint of _shift: W[j + dj, i + di] += Y[j, i]."""
    return _shift(Y, -di, -dj)


def ahat_apply(ga, dc, X):
    """(A_hat x)(a) = A_a x_a + sum_d C_{a,d} x_{a+d}   (kkt_assembly.py:59-64, 217-246)."""
    Y = np.einsum("jiab,jib->jia", ga.A[dc], X)
    for d, (di, dj) in enumerate(_DIRS):
        Y = Y + np.einsum("jiab,jib->jia", ga.C[dc, d], _shift(X, di, dj))
    return Y


def ahat_apply_t(ga, dc, Y):
    """A_hat' y (kkt_assembly.py:66-71)."""
    Z = np.einsum("jiba,jib->jia", ga.A[dc], Y)
    for d, (di, dj) in enumerate(_DIRS):
        Z = Z + _unshift(np.einsum("jiba,jib->jia", ga.C[dc, d], Y), di, dj)
    return Z


def _stages(ga, v, width):
    return np.asarray(v, dtype=float).reshape(-1, ga.N, ga.K, width)


def constraint_t(ga, lam):
    """A~' lam: -lam_t + A_hat_t' lam_{t+1} (kkt_assembly.py:97-105)."""
    L = _stages(ga, lam, ga.n)
    out = -L.copy()
    for t in range(ga.T):
        out[t] += ahat_apply_t(ga, ga.dyn_class[t], L[t + 1])
    return out


def recover(ga, lam):
    """x = -Qinv (A~' lam), u = -Rinv (B~' lam), objective (recovery.py:50-65)."""
    a = constraint_t(ga, lam)
    L = _stages(ga, lam, ga.n)
    qinv = np.linalg.inv(ga.Q)
    rinv = np.linalg.inv(ga.R)
    x = np.stack([-np.einsum("jiab,jib->jia", qinv[ga.cost_class[t]], a[t])
                  for t in range(ga.T + 1)])
    u = np.stack([-np.einsum("jiab,jib->jia", rinv[ga.dyn_class[t]],
                             np.einsum("jiba,jib->jia", ga.B[ga.dyn_class[t]], L[t + 1]))
                  for t in range(ga.T)])
    obj = 0.0
    for t in range(ga.T + 1):
        obj += float(np.sum(x[t] * np.einsum("jiab,jib->jia", ga.Q[ga.cost_class[t]], x[t])))
    for t in range(ga.T):
        obj += float(np.sum(u[t] * np.einsum("jiab,jib->jia", ga.R[ga.dyn_class[t]], u[t])))
    return x.reshape(-1), u.reshape(-1), 0.5 * obj


def kkt(ga, lam, x, u):
    """(||Qx + A~'lam||, ||Ru + B~'lam||, ||A~x + B~u + omega~||) (recovery.py:68-80)."""
    a = constraint_t(ga, lam)
    L = _stages(ga, lam, ga.n)
    X = _stages(ga, x, ga.n)
    U = _stages(ga, u, ga.m)
    off = _stages(ga, ga.offset, ga.n)
    rx = np.stack([np.einsum("jiab,jib->jia", ga.Q[ga.cost_class[t]], X[t]) + a[t]
                   for t in range(ga.T + 1)])
    ru = np.stack([np.einsum("jiab,jib->jia", ga.R[ga.dyn_class[t]], U[t])
                   + np.einsum("jiba,jib->jia", ga.B[ga.dyn_class[t]], L[t + 1])
                   for t in range(ga.T)])
    rd = -X + off
    for t in range(ga.T):
        dc = ga.dyn_class[t]
        rd[t + 1] += ahat_apply(ga, dc, X[t]) + np.einsum("jiab,jib->jia", ga.B[dc], U[t])
    inf = lambda v: float(np.max(np.abs(v))) if v.size else 0.0
    return inf(rx), inf(ru), inf(rd)
