"""Oracle pins: Green's function, quadrature, Lagrange basis, static potentials,
RWG geometry.  Each pin is something other than the oracle itself: values
SPEC.md prints, closed-form integrals, brute-force adaptive quadrature."""
import math
import os

import numpy as np
import pytest
from scipy import integrate

from oracle.green import green, green_grid, green_smooth
from oracle.geometry import dunavant7, triangle_quadrature, rwg_geometry, validate_mesh, MeshError
from oracle.potentials import static_potentials
from oracle.aim import lagrange
from workloads import make_mesh, cube_surface

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_green_golden_values():
    rows = [l.split() for l in open(os.path.join(GOLDEN, "green_values.txt")) if l.strip() and not l.startswith("#")]
    for R, k, mag, ph, *_ in rows:
        g = complex(green(float(R), float(k)))
        assert abs(abs(g) - float(mag)) < 5e-8
        d = (np.angle(g) - float(ph) + math.pi) % (2 * math.pi) - math.pi
        assert abs(d) < 1e-12


def test_green_smooth_and_grid():
    k = 2 * math.pi
    R = np.array([1e-3, 0.05, 0.3, 1.7])
    np.testing.assert_allclose(green_smooth(R, k) + 1 / (4 * math.pi * R), green(R, k), rtol=1e-13)
    # limit at 0: (exp(-jkR)-1)/(4 pi R) -> -jk/(4 pi); Taylor: -jk/4pi - k^2 R/8pi
    r0 = 1e-7
    assert abs(green_smooth(np.array([r0]), k)[0] - (-1j * k / (4 * math.pi) - k * k * r0 / (8 * math.pi))) < 1e-12
    assert green_smooth(np.array([0.0]), k)[0] == -1j * k / (4 * math.pi)
    assert green_grid(np.array([0.0, 0.5]), k)[0] == 0
    assert green_grid(np.array([0.0, 0.5]), k)[1] == green(0.5, k)


def test_dunavant_exact_to_degree_5():
    bary, w = dunavant7()
    assert abs(w.sum() - 1) < 1e-15
    assert (bary > 0).all() and np.allclose(bary.sum(1), 1)
    # reference triangle (0,0),(1,0),(0,1), area 1/2: int x^a y^b = a! b!/(a+b+2)!
    x, y = bary[:, 1], bary[:, 2]
    for a in range(7):
        for b in range(7 - a):
            exact = math.factorial(a) * math.factorial(b) / math.factorial(a + b + 2)
            q = 0.5 * np.sum(w * x ** a * y ** b)
            if a + b <= 5:
                assert abs(q - exact) < 1e-15, (a, b)
    # degree 6 is NOT integrated exactly (it is a degree-5 rule)
    assert abs(0.5 * np.sum(w * x ** 6) - math.factorial(6) / math.factorial(8)) > 1e-6


def test_lagrange_basis():
    for M in (1, 2, 3, 4):
        L = lagrange(np.arange(M + 1, dtype=float), M)
        np.testing.assert_array_equal(L, np.eye(M + 1))
        t = np.linspace(-0.7, M + 0.3, 29)
        Lt = lagrange(t, M)
        for p in range(M + 1):  # reproduces all polynomials of degree <= M
            np.testing.assert_allclose(Lt @ (np.arange(M + 1) ** p), t ** p, atol=1e-11)


TRI = np.array([[0.0, 0.0, 0.0], [1.0, 0.1, 0.0], [0.2, 0.9, 0.0]])


def _brute_potentials(r):
    v1, v2, v3 = TRI
    J = np.linalg.norm(np.cross(v2 - v1, v3 - v1))
    out = []
    for comp in (-1, 0, 1, 2):
        def f(t, s):
            p = v1 + s * (v2 - v1) + t * (v3 - v1)
            return (1.0 if comp < 0 else p[comp]) / np.linalg.norm(r - p) * J
        out.append(integrate.dblquad(f, 0, 1, 0, lambda s: 1 - s, epsabs=1e-13, epsrel=1e-12)[0])
    return np.array(out)


@pytest.mark.parametrize("r", [
    [0.3, 0.3, 0.5],        # off-plane above interior
    [0.3, 0.3, 1e-4],       # nearly in-plane, interior
    [2.0, -1.0, 0.3],       # far, off-plane
    [-0.5, 0.05, 0.0],      # in-plane, outside
    [1.5, 0.15, 0.0],       # in-plane on the extension of edge v1->v2 (edge-line guard)
    [0.4, 0.04, 0.2],       # above an edge
])
def test_static_potentials_vs_adaptive(r):
    r = np.array(r)
    I0, Ir = static_potentials(r[None], TRI[None])
    b = _brute_potentials(r)
    assert abs(I0[0] - b[0]) <= 1e-6 * abs(b[0])
    assert np.all(np.abs(Ir[0] - b[1:]) <= 1e-6 * np.abs(b[1:]).max())


def test_rwg_geometry_invariants():
    m = make_mesh("c1")
    validate_mesh(m.vertices, m.triangles, m.rwg)
    g = rwg_geometry(m.vertices, m.triangles, m.rwg)
    # normal component of Lambda across the edge is 1 on both sides (RWG definition)
    v = m.vertices
    va, vb = v[m.rwg[:, 0]], v[m.rwg[:, 1]]
    mid = 0.5 * (va + vb)
    e = (vb - va) / g["l"][:, None]
    for p, A, sgn in ((g["pp"], g["Ap"], 1.0), (g["pm"], g["Am"], -1.0)):
        lam = sgn * g["l"][:, None] / (2 * A[:, None]) * (mid - p)
        # in-plane normal of the edge pointing away from the free vertex
        d = mid - p
        un = d - (d * e).sum(1)[:, None] * e
        un /= np.linalg.norm(un, axis=1)[:, None]
        flux = (lam * un).sum(1)
        np.testing.assert_allclose(flux, sgn * np.ones_like(flux), rtol=1e-12)
    # charge neutrality: int div Lambda = l - l = 0 (areas x divergences)
    np.testing.assert_allclose(g["l"] / g["Ap"] * g["Ap"] - g["l"] / g["Am"] * g["Am"], 0, atol=1e-15)


def test_validate_mesh_errors():
    m = cube_surface((0, 0, 0), 1.0, 2)
    bad = m.rwg.copy()
    bad[0, 3] = bad[0, 2]
    with pytest.raises(MeshError):
        validate_mesh(m.vertices, m.triangles, bad)
    bad = m.rwg.copy()
    bad[0, 0] = (bad[0, 0] + 5) % m.vertices.shape[0]
    with pytest.raises(MeshError):
        validate_mesh(m.vertices, m.triangles, bad)
    t = m.triangles.copy()
    t[0, 1] = t[0, 0]
    with pytest.raises(MeshError):
        validate_mesh(m.vertices, t, m.rwg)


def test_quadrature_areas():
    m = make_mesh("c1")
    pts, wts = triangle_quadrature(m.vertices, m.triangles)
    # each cube surface area 6 * 0.4^2
    np.testing.assert_allclose(wts.sum(), 4 * 6 * 0.16, rtol=1e-13)
