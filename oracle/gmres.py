"""Restarted GMRES ("we solve the linear system ...
iteratively using the generalized minimal residual (GMRES) algorithm"),
reading D15:

  * x0 = 0; Arnoldi with modified Gram-Schmidt plus one reorthogonalisation
    pass; complex Givens rotations on the Hessenberg matrix;
  * stop when the residual estimate |g_{j+1}| / ||b|| <= tol; at the end of
    a cycle (or on the estimate) the true residual is recomputed and the
    iteration continues (restart) if it is above tol;
  * non-convergence within max_iters is a flag, never an exception;
  * `fixed_iters` runs exactly that many inner iterations (the parity
    protocol "at equal iteration counts") and returns the iterate.
"""
from __future__ import annotations

import numpy as np


def _givens(a, b):
    if a == 0:
        return 0.0, 1.0 + 0j
    r = np.sqrt(abs(a) ** 2 + abs(b) ** 2)
    c = abs(a) / r
    s = (a / abs(a)) * np.conj(b) / r
    return c, s


def gmres(matvec, b, restart=50, tol=1e-4, max_iters=20000, fixed_iters=None):
    b = np.asarray(b, dtype=np.complex128)
    n = b.size
    x = np.zeros(n, dtype=np.complex128)
    bnorm = np.linalg.norm(b)
    hist = []
    if bnorm == 0:
        return dict(x=x, iters=0, rel_res=0.0, converged=True, history=hist)
    total = 0
    limit = fixed_iters if fixed_iters is not None else max_iters
    r = b.copy()
    beta = bnorm
    while True:
        V = np.zeros((restart + 1, n), dtype=np.complex128)
        H = np.zeros((restart + 1, restart), dtype=np.complex128)
        cs = np.zeros(restart)
        sn = np.zeros(restart, dtype=np.complex128)
        g = np.zeros(restart + 1, dtype=np.complex128)
        g[0] = beta
        V[0] = r / beta
        j_done = 0
        stop = False
        for j in range(restart):
            w = matvec(V[j])
            for _ in range(2):                      # MGS + one reorthogonalisation
                for i in range(j + 1):
                    hij = np.vdot(V[i], w)
                    H[i, j] += hij
                    w = w - hij * V[i]
            hn = np.linalg.norm(w)
            H[j + 1, j] = hn
            if hn > 0:
                V[j + 1] = w / hn
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -np.conj(sn[i]) * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            c, s = _givens(H[j, j], H[j + 1, j])
            cs[j], sn[j] = c, s
            H[j, j] = c * H[j, j] + s * H[j + 1, j]
            H[j + 1, j] = 0.0
            g[j + 1] = -np.conj(s) * g[j]
            g[j] = c * g[j]
            total += 1
            j_done = j + 1
            est = abs(g[j + 1]) / bnorm
            hist.append(est)
            if total >= limit:
                stop = True
                break
            if fixed_iters is None and est <= tol:
                break
            if hn == 0:
                break
        y = np.linalg.solve(np.triu(H[:j_done, :j_done]), g[:j_done]) if j_done else np.zeros(0)
        x = x + V[:j_done].T @ y
        r = b - matvec(x)
        beta = np.linalg.norm(r)
        rel = beta / bnorm
        if stop or (fixed_iters is None and rel <= tol) or beta == 0:
            conv = rel <= tol
            return dict(x=x, iters=total, rel_res=rel, converged=bool(conv), history=hist)
