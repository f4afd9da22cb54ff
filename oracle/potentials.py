"""Analytic static potential integrals over a flat triangle (D8).

For observation point r and triangle t' = (v1, v2, v3) with unit normal
n = (v2-v1)x(v3-v1)/|.|, d = n.(r - v1), rho = r - d n.  For each directed
edge a->b (v1->v2, v2->v3, v3->v1):
    lhat = (b-a)/|b-a|,  u = lhat x n (outward in-plane edge normal)
    l+ = (b-rho).lhat,  l- = (a-rho).lhat,  P0 = (a-rho).u  (signed)
    R0^2 = P0^2 + d^2,  R+ = |r-b|,  R- = |r-a|
    f = ln((R+ + l+)/(R- + l-))   (0 on the edge line R0 = 0)
I0 = int 1/R dS' = sum [P0 f - |d|(atan2(P0 l+, R0^2+|d|R+) - atan2(P0 l-, R0^2+|d|R-))]
I1 = int (rho'-rho)/R dS' = 1/2 sum u [R0^2 f + l+ R+ - l- R-]
int r'/R dS' = I1 + rho I0.
(Standard potential-integral formulas for a flat triangle, as restated in
SURVEY.md §8(c) "Closed forms"; pinned in tests against adaptive subdivision.)
For l < 0 the stable form R + l = R0^2/(R - l) is used.
"""
from __future__ import annotations

import numpy as np


def _r_plus_l(R, l, R0sq):
    out = np.empty_like(R)
    pos = l >= 0
    out[pos] = R[pos] + l[pos]
    neg = ~pos
    out[neg] = R0sq[neg] / (R[neg] - l[neg])
    return out


def static_potentials(r, corners):
    """r: (K,3) observation points; corners: (K,3,3) triangle vertices.

    Returns I0 (K,) = int 1/R dS' and Ir (K,3) = int r'/R dS'.
    """
    r = np.asarray(r, dtype=np.float64)
    c = np.asarray(corners, dtype=np.float64)
    v1, v2, v3 = c[:, 0], c[:, 1], c[:, 2]
    cr = np.cross(v2 - v1, v3 - v1)
    n = cr / np.linalg.norm(cr, axis=1)[:, None]
    d = np.einsum("kd,kd->k", n, r - v1)
    rho = r - d[:, None] * n
    ad = np.abs(d)
    I0 = np.zeros(r.shape[0])
    I1 = np.zeros((r.shape[0], 3))
    for a, b in ((v1, v2), (v2, v3), (v3, v1)):
        e = b - a
        le = np.linalg.norm(e, axis=1)
        lhat = e / le[:, None]
        u = np.cross(lhat, n)
        lp = np.einsum("kd,kd->k", b - rho, lhat)
        lm = np.einsum("kd,kd->k", a - rho, lhat)
        P0 = np.einsum("kd,kd->k", a - rho, u)
        R0sq = P0 * P0 + d * d
        Rp = np.linalg.norm(r - b, axis=1)
        Rm = np.linalg.norm(r - a, axis=1)
        on_line = R0sq <= (1e-12 * le) ** 2
        f = np.zeros_like(R0sq)
        ok = ~on_line
        if ok.any():
            num = _r_plus_l(Rp[ok], lp[ok], R0sq[ok])
            den = _r_plus_l(Rm[ok], lm[ok], R0sq[ok])
            f[ok] = np.log(num / den)
        I0 += P0 * f - ad * (np.arctan2(P0 * lp, R0sq + ad * Rp) - np.arctan2(P0 * lm, R0sq + ad * Rm))
        I1 += 0.5 * u * (R0sq * f + lp * Rp - lm * Rm)[:, None]
    Ir = I1 + rho * I0[:, None]
    return I0, Ir
