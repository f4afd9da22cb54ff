"""Oracle pins: plane-wave RHS and GMRES (D14, D15)."""
import numpy as np
import pytest
import scipy.sparse as sp

from conftest import oracle_plan
from oracle.constants import ETA0
from oracle.excitation import plane_wave_field, plane_wave_rhs
from oracle.gmres import gmres


def test_plane_wave_field_values():
    k = 2 * np.pi
    E = plane_wave_field(np.array([[0.0, 0.0, 0.0], [0.0, 0.0, 0.25], [3.0, -1.0, 0.5]]), k)
    np.testing.assert_allclose(E[0], [1, 0, 0])
    np.testing.assert_allclose(E[1], [1j, 0, 0], atol=1e-15)    # exp(+j k z), z = lambda/4
    np.testing.assert_allclose(E[2], [-1, 0, 0], atol=1e-15)


def test_plane_wave_rhs_bruteforce_and_linearity():
    P = oracle_plan("c1")
    V = plane_wave_rhs(P.ctx)
    V2 = plane_wave_rhs(P.ctx, E0=2.5 - 1j)
    np.testing.assert_allclose(V2, (2.5 - 1j) * V, rtol=1e-14)
    # brute force: 4^3 sub-triangles x 7-point rule on both RWG triangles
    ctx = P.ctx
    from oracle.geometry import dunavant7
    bary, w = dunavant7()

    def sub(tri, lev):
        if lev == 0:
            return [tri]
        a, b, c = tri
        ab, bc, ca = (a + b) / 2, (b + c) / 2, (c + a) / 2
        out = []
        for t in ((a, ab, ca), (ab, b, bc), (ca, bc, c), (ab, bc, ca)):
            out += sub(np.array(t), lev - 1)
        return out

    for n in (0, 100, 777):
        tot = 0j
        for side in (0, 1):
            t = ctx.side_tri[n, side]
            al, p = ctx.side_alpha[n, side], ctx.side_p[n, side]
            for st in sub(ctx.tgeo["corners"][t], 3):
                A = 0.5 * np.linalg.norm(np.cross(st[1] - st[0], st[2] - st[0]))
                r = bary @ st
                E = plane_wave_field(r, P.k)
                tot += np.sum(w * A * np.einsum("qd,qd->q", al * (r - p), E))
        assert abs(tot - V[n]) <= 1e-5 * abs(tot)


def test_gmres_identity_and_diag():
    b = np.array([1.0 + 2j, -3.0, 0.5j])
    res = gmres(lambda v: v, b, restart=5, tol=1e-12)
    assert res["iters"] == 1 and np.allclose(res["x"], b) and res["converged"]
    D = np.array([2.0, 3.0])
    res = gmres(lambda v: D * v, np.array([2.0, 3.0]), restart=5, tol=1e-12)
    assert res["iters"] <= 2 and np.allclose(res["x"], [1, 1], atol=1e-12)
    res = gmres(lambda v: D * v, np.zeros(2), restart=5, tol=1e-12)
    assert res["iters"] == 0 and not res["x"].any()


def test_gmres_not_converged_is_flag():
    rng = np.random.default_rng(0)
    A = rng.standard_normal((40, 40)) + 1j * rng.standard_normal((40, 40))
    b = rng.standard_normal(40) + 0j
    res = gmres(lambda v: A @ v, b, restart=3, tol=1e-14, max_iters=7)
    assert not res["converged"] and res["iters"] == 7


def test_gmres_matches_dense_solve_c1():
    """C1: GMRES on the AIM operator vs LU of the explicitly formed Z_eq."""
    P = oracle_plan("c1")
    Pm = P.projection_matrices()
    H = P.kernel_matrix()
    far = sum((Pm[c].T @ (H @ Pm[c].toarray())) for c in range(3)) - (Pm[3].T @ (H @ Pm[3].toarray())) / P.k ** 2
    Z = 1j * P.k * ETA0 * far + P.near_full().toarray()
    x = np.random.default_rng(1).standard_normal(P.N) + 0j
    assert np.linalg.norm(Z @ x - P.matvec(x)) <= 1e-12 * np.linalg.norm(Z @ x)
    V = plane_wave_rhs(P.ctx)
    ref = np.linalg.solve(Z, V)
    res = gmres(lambda v: Z @ v, V, restart=50, tol=1e-8, max_iters=3000)
    assert res["converged"] and res["rel_res"] <= 1e-8
    kappa = np.linalg.cond(Z)
    assert np.linalg.norm(res["x"] - ref) <= 1e-8 * kappa * np.linalg.norm(ref)
    # monotone residual estimate within each cycle, deterministic history
    h = np.array(res["history"])
    for c in range(0, h.size, 50):
        seg = h[c:c + 50]
        assert (np.diff(seg) <= 1e-15).all()
    res2 = gmres(lambda v: Z @ v, V, restart=50, tol=1e-8, max_iters=3000)
    assert res2["history"] == res["history"]
