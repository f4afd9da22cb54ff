"""Plane-wave right-hand side (reading D1/D14).

V_m = <Lambda_m, E_inc> = sum_{t in T_m} sum_q w_q Lambda_m(r_q) . E_inc(r_q)
(7-point rule, D7), with E_inc(r) = E0 pol exp(-j k khat.r)  (e^{+j omega t}).
The paper's V-hat = <Lambda, n x n x E_inc> = -<Lambda, E_inc_tan>; with the
sign convention of D1 (Z = -G) the solved system is Z J = V with V as above.
Config 4: khat = -z, pol = x, E0 = 1  ->  E_inc = x exp(+j k z).
"""
from __future__ import annotations

import numpy as np

from .efie import EfieContext


def plane_wave_field(r, k, khat=(0.0, 0.0, -1.0), pol=(1.0, 0.0, 0.0), E0=1.0):
    r = np.asarray(r, dtype=np.float64)
    ph = np.exp(-1j * k * (r @ np.asarray(khat, dtype=np.float64)))
    return E0 * ph[..., None] * np.asarray(pol, dtype=np.float64)


def plane_wave_rhs(ctx: EfieContext, khat=(0.0, 0.0, -1.0), pol=(1.0, 0.0, 0.0), E0=1.0):
    N = ctx.rwg.shape[0]
    V = np.zeros(N, dtype=np.complex128)
    for side in (0, 1):
        t = ctx.side_tri[:, side]
        a = ctx.side_alpha[:, side]
        p = ctx.side_p[:, side]
        rq = ctx.qpts[t]                               # (N,7,3)
        wq = ctx.qw[t]
        lam = a[:, None, None] * (rq - p[:, None, :])  # (N,7,3)
        E = plane_wave_field(rq, ctx.k, khat, pol, E0)
        V += np.einsum("nq,nqd,nqd->n", wq, lam, E)
    return V
