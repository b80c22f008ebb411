"""Prototype: exact domain-decomposed solve of an SPD block-tridiagonal chain (separator
blocks every m blocks), checked against the plain block-LDL^T recurrence."""
import numpy as np

rng = np.random.default_rng(0)
q, nb, m = 8, 37, 8


def spd_chain():
    D = [None] * nb
    E = [None] * nb
    for k in range(nb):
        a = rng.standard_normal((q, q))
        D[k] = a @ a.T + 3 * q * np.eye(q)
        if k:
            E[k] = rng.standard_normal((q, q))
    return D, E


def dense(D, E, lo, hi):
    n = hi - lo
    A = np.zeros((n * q, n * q))
    for k in range(lo, hi):
        i = k - lo
        A[i*q:(i+1)*q, i*q:(i+1)*q] = D[k]
        if k > lo:
            A[i*q:(i+1)*q, (i-1)*q:i*q] = E[k]
            A[(i-1)*q:i*q, i*q:(i+1)*q] = E[k].T
    return A


def factor(D, E, blocks):
    """block Cholesky along `blocks` (consecutive); returns Linv[k], C[k] (C[first]=0)."""
    Linv, C = {}, {}
    prev = None
    for k in blocks:
        S = D[k].copy()
        if prev is not None:
            C[k] = E[k] @ Linv[prev].T
            S = S - C[k] @ C[k].T
        else:
            C[k] = np.zeros((q, q))
        Linv[k] = np.linalg.inv(np.linalg.cholesky(S))
        prev = k
    return Linv, C


def solve(Linv, C, blocks, b):
    w = {}
    prev = None
    for k in blocks:
        s = b[k] if prev is None else b[k] - C[k] @ w[prev]
        w[k] = Linv[k] @ s
        prev = k
    x = {}
    nxt = None
    for k in reversed(blocks):
        s = w[k] if nxt is None else w[k] - C[nxt].T @ x[nxt]
        x[k] = Linv[k].T @ s
        nxt = k
    return x


D, E = spd_chain()
A = dense(D, E, 0, nb)
b = rng.standard_normal((nb, q, 3))          # 3 right-hand sides (chains)
x_ref = np.linalg.solve(A, b.reshape(nb * q, 3)).reshape(nb, q, 3)

# plain recurrence (what the kernels do today)
L0, C0 = factor(D, E, list(range(nb)))
x0 = solve(L0, C0, list(range(nb)), {k: b[k] for k in range(nb)})
print("plain LDL^T  err", max(np.abs(x0[k] - x_ref[k]).max() for k in range(nb)))

# ---- domain decomposition -------------------------------------------------------
ns = (nb + m - 1) // m
seps = [s * m + m - 1 for s in range(ns - 1) if s * m + m - 1 < nb - 1]
ns = len(seps) + 1
interiors = []
lo = 0
for g in seps + [nb]:
    interiors.append(list(range(lo, g)))
    lo = g + 1
assert sum(len(I) for I in interiors) + len(seps) == nb

# setup: interior factors, spikes, separator Schur complement
fac = [factor(D, E, I) for I in interiors]
V, W = [], []
for s, I in enumerate(interiors):
    Ls, Cs = fac[s]
    z = {k: np.zeros((q, q)) for k in I}
    if s > 0:                      # coupling of the first interior block to separator s-1
        zz = dict(z); zz[I[0]] = E[I[0]]
        V.append(solve(Ls, Cs, I, zz))
    else:
        V.append(None)
    if s < ns - 1:                 # coupling of the last interior block to separator s
        zz = dict(z); zz[I[-1]] = E[seps[s]].T
        W.append(solve(Ls, Cs, I, zz))
    else:
        W.append(None)
Sd, Ssub = [], []
for s, g in enumerate(seps):
    Sss = D[g] - E[g] @ W[s][interiors[s][-1]] - E[interiors[s + 1][0]].T @ V[s + 1][interiors[s + 1][0]]
    Sd.append(Sss)
    if s > 0:
        # S[s][s-1] = - A[g_s, I_s] A_II^-1 A[I_s, g_{s-1}] = - E[g_s] V_s[last]
        Ssub.append(-E[g] @ V[s][interiors[s][-1]])
    else:
        Ssub.append(None)
Sfac = factor(Sd, [None] + Ssub[1:], list(range(len(seps))))

# solve
u = [solve(fac[s][0], fac[s][1], I, {k: b[k] for k in I}) for s, I in enumerate(interiors)]
g_rhs = {}
for s, g in enumerate(seps):
    g_rhs[s] = b[g] - E[g] @ u[s][interiors[s][-1]] - E[interiors[s + 1][0]].T @ u[s + 1][interiors[s + 1][0]]
xg = solve(Sfac[0], Sfac[1], list(range(len(seps))), g_rhs)
x = {}
for s, I in enumerate(interiors):
    for k in I:
        v = u[s][k]
        if s > 0:
            v = v - V[s][k] @ xg[s - 1]
        if s < ns - 1:
            v = v - W[s][k] @ xg[s]
        x[k] = v
for s, g in enumerate(seps):
    x[g] = xg[s]
print("domain-decomposed err", max(np.abs(x[k] - x_ref[k]).max() for k in range(nb)))
