"""Exact Galerkin EFIE entries of the exterior operator (the paper's G^(E^,J^)).

PAPER.md:460-472 (eq. Gouter1): entry = j omega mu0 <Lambda_m, n x n x L Lambda_n>
with L X = (1 + k^-2 grad div) int G X.  Reading D1
(SURVEY.md §8(c)): the operator of the solved system Z J = V is the
mixed-potential form

    Z_mn = j k eta0 int_{T_m} int_{T_n} G(|r-r'|) [Lambda_m(r).Lambda_n(r')
                                   - k^-2 div Lambda_m(r) div' Lambda_n(r')] dS' dS

(j omega mu0 = j k eta0), evaluated per triangle pair (t, t') through the
moments  I00 = int int G,  I10 = int int G r,  I01 = int int G r',
I11 = int int G r.r'.  With Lambda_m = alpha (r - p_m) on t and
Lambda_n = beta (r' - p_n) on t' (geometry.py), the pair contributes

    j k eta0 ( alpha beta [I11 - p_n.I10 - p_m.I01 + (p_m.p_n) I00]
               - k^-2 (2 alpha)(2 beta) I00 ).

Quadrature (D7, D8): 7x7 product rule, except for triangle pairs sharing at
least one vertex index, where the inner integral is
    sum_p w_p G_s(R_qp) {1, r_p} + (1/4 pi) {I0(r_q), Ir(r_q)}
(green.green_smooth + potentials.static_potentials).  Symmetrisation (D9):
Z_ex_sym = (Z_ex + Z_ex^T)/2.
"""
from __future__ import annotations

import numpy as np

from .constants import ETA0
from .geometry import triangle_quadrature, rwg_geometry, triangle_geometry
from .green import green, green_smooth
from .potentials import static_potentials


class EfieContext:
    """Per-mesh data for the exact entries (quadrature, RWG geometry)."""

    def __init__(self, vertices, triangles, rwg, k):
        self.vertices = np.asarray(vertices, dtype=np.float64)
        self.triangles = np.asarray(triangles, dtype=np.int64)
        self.rwg = np.asarray(rwg, dtype=np.int64)
        self.k = float(k)
        self.qpts, self.qw = triangle_quadrature(self.vertices, self.triangles)
        self.geo = rwg_geometry(self.vertices, self.triangles, self.rwg)
        self.tgeo = triangle_geometry(self.vertices, self.triangles)
        g = self.geo
        # per RWG, per side s in (+, -): triangle, alpha = sigma l/(2A), free vertex
        self.side_tri = np.stack([g["tp"], g["tm"]], axis=1)
        self.side_alpha = np.stack([g["l"] / (2 * g["Ap"]), -g["l"] / (2 * g["Am"])], axis=1)
        self.side_p = np.stack([g["pp"], g["pm"]], axis=1)


def share_vertex(triangles, t, tp):
    """True where triangles t and tp share at least one vertex index (D8)."""
    a = triangles[t]
    b = triangles[tp]
    return (a[:, :, None] == b[:, None, :]).any(axis=(1, 2))


def tri_pair_moments(ctx: EfieContext, t, tp, chunk=20000):
    """Moments (I00, I10, I01, I11) for triangle pairs (t[i] test, tp[i] source)."""
    t = np.asarray(t, dtype=np.int64)
    tp = np.asarray(tp, dtype=np.int64)
    K = t.size
    I00 = np.zeros(K, dtype=np.complex128)
    I10 = np.zeros((K, 3), dtype=np.complex128)
    I01 = np.zeros((K, 3), dtype=np.complex128)
    I11 = np.zeros(K, dtype=np.complex128)
    sing = share_vertex(ctx.triangles, t, tp)
    k = ctx.k
    for s in range(0, K, chunk):
        sl = slice(s, min(K, s + chunk))
        ti, tj, sg = t[sl], tp[sl], sing[sl]
        rq = ctx.qpts[ti]            # (c,7,3) outer points
        wq = ctx.qw[ti]              # (c,7)
        rp = ctx.qpts[tj]            # (c,7,3) inner points
        wp = ctx.qw[tj]
        R = np.linalg.norm(rq[:, :, None, :] - rp[:, None, :, :], axis=3)  # (c,7,7)
        # regular 7x7 rule
        Gf = np.where(sg[:, None, None], 0.0, 1.0) * green(np.where(R > 0, R, 1.0), k)
        Gs = np.where(sg[:, None, None], 1.0, 0.0) * green_smooth(R, k)
        Gk = Gf + Gs                                     # G (regular) or G_s (singular)
        in0 = np.einsum("cqp,cp->cq", Gk, wp)            # inner int of G   (c,7)
        in1 = np.einsum("cqp,cp,cpd->cqd", Gk, wp, rp)   # inner int of G r' (c,7,3)
        if sg.any():
            idx = np.nonzero(sg)[0]
            corners = ctx.tgeo["corners"][tj[idx]]       # (s,3,3)
            obs = rq[idx].reshape(-1, 3)
            cor = np.repeat(corners, 7, axis=0)
            J0, Jr = static_potentials(obs, cor)
            in0[idx] += (J0.reshape(-1, 7)) / (4 * np.pi)
            in1[idx] += (Jr.reshape(-1, 7, 3)) / (4 * np.pi)
        I00[sl] = np.einsum("cq,cq->c", wq, in0)
        I10[sl] = np.einsum("cq,cq,cqd->cd", wq, in0, rq)
        I01[sl] = np.einsum("cq,cqd->cd", wq, in1)
        I11[sl] = np.einsum("cq,cqd,cqd->c", wq, rq, in1)
    return I00, I10, I01, I11


def _combine(ctx, k, a, b, pm, pn, I00, I10, I01, I11):
    lam = a * b * (I11 - np.einsum("kd,kd->k", pn, I10) - np.einsum("kd,kd->k", pm, I01)
                   + np.einsum("kd,kd->k", pm, pn) * I00)
    chg = (2 * a) * (2 * b) * I00 / (k * k)
    return 1j * k * ETA0 * (lam - chg)


def efie_entries(ctx: EfieContext, m, n):
    """Z_ex[m, n] (unsymmetrised) for RWG pairs given as index arrays.

    The moments of each distinct triangle pair are computed once and
    gathered (a triangle pair serves up to 3x3 RWG pairs)."""
    m = np.asarray(m, dtype=np.int64)
    n = np.asarray(n, dtype=np.int64)
    nt = ctx.triangles.shape[0]
    keys = np.concatenate([ctx.side_tri[m, sm] * nt + ctx.side_tri[n, sn]
                           for sm in (0, 1) for sn in (0, 1)])
    uniq, inv = np.unique(keys, return_inverse=True)
    I00, I10, I01, I11 = tri_pair_moments(ctx, uniq // nt, uniq % nt)
    out = np.zeros(m.size, dtype=np.complex128)
    for c, (sm, sn) in enumerate((a, b) for a in (0, 1) for b in (0, 1)):
        g = inv[c * m.size:(c + 1) * m.size]
        out += _combine(ctx, ctx.k, ctx.side_alpha[m, sm], ctx.side_alpha[n, sn],
                        ctx.side_p[m, sm], ctx.side_p[n, sn], I00[g], I10[g], I01[g], I11[g])
    return out


def efie_entries_sym(ctx: EfieContext, m, n):
    """Z_ex_sym[m, n] = (Z_ex[m,n] + Z_ex[n,m]) / 2   (D9)."""
    return 0.5 * (efie_entries(ctx, m, n) + efie_entries(ctx, n, m))


def dense_Z(ctx: EfieContext):
    """Full symmetrised exact matrix (tiny meshes only: O(N^2) memory)."""
    N = ctx.rwg.shape[0]
    nt = ctx.triangles.shape[0]
    tt, ss = np.meshgrid(np.arange(nt), np.arange(nt), indexing="ij")
    I00, I10, I01, I11 = tri_pair_moments(ctx, tt.ravel(), ss.ravel())
    I00 = I00.reshape(nt, nt)
    I10 = I10.reshape(nt, nt, 3)
    I01 = I01.reshape(nt, nt, 3)
    I11 = I11.reshape(nt, nt)
    k = ctx.k
    Z = np.zeros((N, N), dtype=np.complex128)
    for sm in (0, 1):
        for sn in (0, 1):
            t = ctx.side_tri[:, sm]
            tp = ctx.side_tri[:, sn]
            a = ctx.side_alpha[:, sm][:, None]
            b = ctx.side_alpha[:, sn][None, :]
            pm = ctx.side_p[:, sm]          # (N,3)
            pn = ctx.side_p[:, sn]
            i00 = I00[np.ix_(t, tp)]
            i10 = I10[t][:, tp]             # (N,N,3)
            i01 = I01[t][:, tp]
            i11 = I11[np.ix_(t, tp)]
            lam = a * b * (i11 - np.einsum("nd,mnd->mn", pn, i10) - np.einsum("md,mnd->mn", pm, i01)
                           + (pm @ pn.T) * i00)
            chg = (2 * a) * (2 * b) * i00 / (k * k)
            Z += 1j * k * ETA0 * (lam - chg)
    return 0.5 * (Z + Z.T)
