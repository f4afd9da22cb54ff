"""Oracle pins for the AIM operator (SURVEY.md §8(c) "What pins each part").

Projection-weight moment identities, convolution (direct sum vs FFT, brute
force, padding independence), near-pair exactness through the FFT far path,
linearity, complex symmetry, translation invariance, dense-MoM agreement,
and exact EFIE entries vs pointwise / subdivided brute force."""
import math

import numpy as np
import pytest
from scipy import integrate

from conftest import oracle_plan
from oracle.aim import OraclePlan, stencil_bases
from oracle.constants import ETA0
from oracle.efie import dense_Z, efie_entries
from oracle.green import green, green_grid
from workloads import make_mesh, make_vectors, get_config
from workloads.meshes import Mesh


def _moments_quadrature(P, n, a, b, c):
    """sum_q w_q f^psi(r_q) x^a y^b z^c directly from the RWG definition."""
    ctx = P.ctx
    out = np.zeros(4)
    for side in (0, 1):
        t = ctx.side_tri[n, side]
        rq, wq = ctx.qpts[t], ctx.qw[t]
        al, p = ctx.side_alpha[n, side], ctx.side_p[n, side]
        mono = rq[:, 0] ** a * rq[:, 1] ** b * rq[:, 2] ** c
        out[:3] += (wq * mono) @ (al * (rq - p))
        out[3] += np.sum(wq * mono * 2 * al)
    return out


@pytest.mark.parametrize("name", ["c1", "t_m3"])
def test_projection_moment_identities(name):
    P = oracle_plan(name)
    M = P.M
    rows = np.arange(0, P.N, max(1, P.N // 40))
    for n in rows:
        nodes = P.h * (P.bases[n] + P.offsets).astype(float)          # (S,3) node positions
        for a in range(M + 1):
            for b in range(M + 1):
                for c in range(M + 1):
                    mono = nodes[:, 0] ** a * nodes[:, 1] ** b * nodes[:, 2] ** c
                    lhs = mono @ P.W[n]
                    rhs = _moments_quadrature(P, n, a, b, c)
                    scale = np.abs(P.W[n]).sum() * np.abs(nodes).max() ** (a + b + c) + 1e-300
                    assert np.all(np.abs(lhs - rhs) <= 1e-12 * scale), (n, a, b, c)
    g = P.ctx.geo
    # (ii) zero net projected charge; (iii) current monopole; (iv) charge dipole
    np.testing.assert_allclose(P.W[:, :, 3].sum(1), 0, atol=1e-12 * np.abs(P.W[:, :, 3]).max())
    cp = P.ctx.tgeo["centroid"][g["tp"]]
    cm = P.ctx.tgeo["centroid"][g["tm"]]
    mono = 0.5 * g["l"][:, None] * (cp - g["pp"]) + 0.5 * g["l"][:, None] * (g["pm"] - cm)
    np.testing.assert_allclose(P.W[:, :, :3].sum(1), mono, atol=1e-13)
    ru = P.h * (P.bases[:, None, :] + P.offsets[None]).astype(float)
    dip = np.einsum("nu,nud->nd", P.W[:, :, 3], ru)
    np.testing.assert_allclose(dip, g["l"][:, None] * (cp - cm), atol=1e-12)
    np.testing.assert_allclose(dip, -mono, atol=1e-12)
    # stencil occupancy: (M+1)^3 nonzeros per function per potential at most
    assert P.W.shape[1] == (M + 1) ** 3


def test_stencil_ties_and_grid_c1():
    P = oracle_plan("c1")
    assert tuple(P.dims) == (12, 12, 7)
    # exact ties are systemic (cube faces grid-aligned): +1e-7 picks the upper node
    assert stencil_bases(np.array([[0.25, -0.25, 0.05]]), 0.1, 2).tolist() == [[2, -3, 0]]
    assert stencil_bases(np.array([[0.3, 0.0, -0.2]]), 0.1, 3).tolist() == [[2, -1, -3]]


def test_convolution_direct_vs_fft_and_bruteforce():
    P = oracle_plan("c1")
    rng = np.random.default_rng(3)
    Q = rng.standard_normal((4,) + tuple(P.dims) + (2,)) + 1j * rng.standard_normal((4,) + tuple(P.dims) + (2,))
    a = P.convolve_direct(Q)
    b = P.convolve_fft(Q)                                        # power-of-two pads
    c = P.convolve_fft(Q, pads=tuple(int(2 * d - 1) for d in P.dims))   # minimal odd pads (D11)
    d = P.convolve_fft(Q, pads=(30, 27, 16))
    for o in (b, c, d):
        assert np.linalg.norm(o - a) <= 1e-13 * np.linalg.norm(a)
    H = P.kernel_matrix()
    assert np.array_equal(H, H.T)
    # brute force with explicit loops on a few output nodes
    Nx, Ny, Nz = P.dims
    for (x, y, z) in [(0, 0, 0), (5, 7, 3), (11, 11, 6)]:
        acc = 0j
        for i in range(Nx):
            for j in range(Ny):
                for k in range(Nz):
                    R = P.h * math.sqrt((x - i) ** 2 + (y - j) ** 2 + (z - k) ** 2)
                    if R > 0:
                        acc += np.exp(-1j * P.k * R) / (4 * math.pi * R) * Q[1, i, j, k, 0]
        assert abs(acc - a[1, x, y, z, 0]) <= 1e-13 * abs(acc)


@pytest.mark.parametrize("name", ["c1", "t_m3"])
def test_near_pairs_exact_through_far_path(name):
    """(near_corrected + grid contribution) = exact entry:
    the far part is evaluated by the FFT path on unit vectors, independently
    of the explicit w^T H w blocks used to precorrect."""
    P = oracle_plan(name)
    near = P.near_full()
    for n in [0, 7, P.N // 2, P.N - 1]:
        e = np.zeros(P.N, dtype=complex)
        e[n] = 1
        col = P.matvec(e, method="fft")
        rows = np.nonzero(np.array(near[:, n].todense()).ravel() != 0)[0]
        ex = P.exact_entries(rows, np.full(rows.size, n))
        assert np.max(np.abs(col[rows] - ex)) <= 1e-12 * np.abs(ex).max()


def test_near_list_definition():
    P = oracle_plan("c1")
    rp, cols = P.near_pairs()
    assert rp[-1] == 172344                                   # SURVEY.md Table D-1
    d = np.linalg.norm(P.centres[np.repeat(np.arange(P.N), np.diff(rp))] - P.centres[cols], axis=1)
    assert d.max() <= P.r * (1 + 1e-9)
    # symmetric list, self pairs included
    S = set(zip(np.repeat(np.arange(P.N), np.diff(rp)).tolist(), cols.tolist()))
    assert all((b, a) in S for (a, b) in list(S)[:5000]) and all((i, i) in S for i in range(P.N))


@pytest.mark.parametrize("name", ["c1", "t_vol"])
def test_operator_linearity_symmetry(name):
    P = oracle_plan(name)
    x = make_vectors(P.N, 2, 0)
    y = make_vectors(P.N, 1, 5)[:, 0]
    Zx = P.matvec(x)
    Zy = P.matvec(y)
    # linearity
    z = P.matvec(2.5 * x[:, 0] - (1 - 3j) * x[:, 1])
    assert np.linalg.norm(z - (2.5 * Zx[:, 0] - (1 - 3j) * Zx[:, 1])) <= 1e-12 * np.linalg.norm(z)
    # complex symmetry x^T Z y = y^T Z x (D9)
    a, b = x[:, 0] @ Zy, y @ Zx[:, 0]
    assert abs(a - b) <= 1e-12 * abs(a)


def test_translation_invariance():
    P = oracle_plan("c1")
    cfg = get_config("c1")
    m = make_mesh(cfg)
    sh = np.array([3, -2, 5]) * cfg.h
    Pt = OraclePlan(Mesh(m.vertices + sh, m.triangles, m.rwg), cfg.k, cfg.h, cfg.M, cfg.near_radius)
    assert np.array_equal(Pt.bases - P.bases, np.tile([3, -2, 5], (P.N, 1)))
    x = make_vectors(P.N, 1, 0)[:, 0]
    y0, y1 = P.matvec(x), Pt.matvec(x)
    assert np.linalg.norm(y1 - y0) <= 1e-12 * np.linalg.norm(y0)


def _efie_pointwise(P, m, n):
    """Z_ex[m,n] by direct 7x7 evaluation of Lambda from the RWG definition."""
    ctx = P.ctx
    k = P.k
    v = ctx.vertices
    va, vb, tp, tm = ctx.rwg[m]
    l_m = np.linalg.norm(v[vb] - v[va])
    vna, vnb, tnp, tnm = ctx.rwg[n]
    l_n = np.linalg.norm(v[vnb] - v[vna])
    tot = 0j
    for t, sm in ((tp, 1.0), (tm, -1.0)):
        A = ctx.tgeo["area"][t]
        free = [q for q in ctx.triangles[t] if q not in (va, vb)][0]
        for tq, sn in ((tnp, 1.0), (tnm, -1.0)):
            B = ctx.tgeo["area"][tq]
            free_n = [q for q in ctx.triangles[tq] if q not in (vna, vnb)][0]
            for r, w in zip(ctx.qpts[t], ctx.qw[t]):
                lam_m = sm * l_m / (2 * A) * (r - v[free])
                for rp, wp in zip(ctx.qpts[tq], ctx.qw[tq]):
                    lam_n = sn * l_n / (2 * B) * (rp - v[free_n])
                    G = green(np.linalg.norm(r - rp), k)
                    tot += w * wp * G * (lam_m @ lam_n - (sm * l_m / A) * (sn * l_n / B) / k ** 2)
    return 1j * k * ETA0 * tot


def test_efie_entries_regular_pointwise():
    P = oracle_plan("c1")
    ctx = P.ctx
    pairs = [(0, 900), (10, 500), (300, 1100), (5, 40)]
    for m, n in pairs:
        tm = set(ctx.triangles[ctx.side_tri[m]].ravel())
        tn = set(ctx.triangles[ctx.side_tri[n]].ravel())
        assert not (tm & tn)
        got = efie_entries(ctx, [m], [n])[0]
        ref = _efie_pointwise(P, m, n)
        assert abs(got - ref) <= 1e-12 * abs(ref)


def _duffy_inner(r, corners, k, n=48):
    """int_{t'} G(|r-r'|) {1, r'} dS' for r in the plane of t': split t' into
    the signed sub-triangles (r, a, b) and integrate each in polar-like
    (Duffy) coordinates, which cancel the 1/R singularity; Gauss-Legendre n x n."""
    x, w = np.polynomial.legendre.leggauss(n)
    x, w = 0.5 * (x + 1), 0.5 * w
    S, T = np.meshgrid(x, x, indexing="ij")
    W = np.outer(w, w)
    nrm = np.cross(corners[1] - corners[0], corners[2] - corners[0])
    nrm /= np.linalg.norm(nrm)
    tot0, tot1 = 0j, np.zeros(3, complex)
    for a, b in ((corners[0], corners[1]), (corners[1], corners[2]), (corners[2], corners[0])):
        d = (a - r)[None, None, :] + T[..., None] * (b - a)[None, None, :]
        cr = np.cross(a - r, b - a) @ nrm                      # signed
        dn = np.linalg.norm(d, axis=2)
        p = r + S[..., None] * d
        f = np.exp(-1j * k * S * dn) / (4 * np.pi * dn) * cr * W
        tot0 += f.sum()
        tot1 += (f[..., None] * p).sum((0, 1))
    return tot0, tot1


@pytest.mark.parametrize("pair", [(17, 17), (17, 18), (40, 41), (40, 42), (40, 48)])
def test_efie_singular_moments_vs_duffy(pair):
    """Vertex-sharing coplanar pairs: moments by singularity subtraction vs
    Duffy-transformed Gauss-Legendre inner integrals (same 7-point outer rule).
    The residual is the 7-point error on the smooth remainder G_s."""
    from oracle.efie import tri_pair_moments, share_vertex
    P = oracle_plan("c1")
    ctx = P.ctx
    t, tp = pair
    assert share_vertex(ctx.triangles, np.array([t]), np.array([tp]))[0]
    assert abs(abs(ctx.tgeo["normal"][t] @ ctx.tgeo["normal"][tp]) - 1) < 1e-12
    I00, I10, I01, I11 = tri_pair_moments(ctx, [t], [tp])
    r0, r1, r11 = 0j, np.zeros(3, complex), 0j
    for r, w in zip(ctx.qpts[t], ctx.qw[t]):
        a, b = _duffy_inner(r, ctx.tgeo["corners"][tp], P.k)
        r0, r1, r11 = r0 + w * a, r1 + w * b, r11 + w * (r @ b)
    assert abs(I00[0] - r0) <= 2e-3 * abs(r0)
    assert np.max(np.abs(I01[0] - r1)) <= 2e-3 * np.abs(r1).max()
    assert abs(I11[0] - r11) <= 2e-3 * abs(r11)


def test_dense_agreement():
    """AIM vs dense MoM <= 1e-3 at h=0.1, M=3, r=0.4 on the C1
    mesh; at C1's own parameters it is a reported number."""
    P3 = oracle_plan("c1", M=3, near_radius=0.4)
    Z = dense_Z(P3.ctx)
    x = make_vectors(P3.N, 1, 0)[:, 0]
    yd = Z @ x
    e3 = np.linalg.norm(P3.matvec(x) - yd) / np.linalg.norm(yd)
    assert e3 <= 1e-3
    P2 = oracle_plan("c1")
    e2 = np.linalg.norm(P2.matvec(x) - yd) / np.linalg.norm(yd)
    assert e2 < 5e-3 and e3 < e2
    # the near part of Z_eq reproduces dense entries exactly on near pairs
    asym = np.linalg.norm(Z - Z.T)
    assert asym == 0


# ------------------------------------------------ the oracle's own FFT (north_star)
@pytest.mark.parametrize("P", [1, 2, 4, 8, 16, 32, 64])
def test_radix2_fft_vs_direct_dft(P):
    """oracle/fft.py radix-2 Cooley-Tukey == the O(P^2) definition, both
    directions, along every axis of a 3-D array; inverse(forward) = identity."""
    from oracle.fft import dft_direct, fft_radix2
    rng = np.random.default_rng(P)
    a = rng.standard_normal((3, P, 5)) + 1j * rng.standard_normal((3, P, 5))
    for inv in (False, True):
        f = fft_radix2(a, axis=1, inverse=inv)
        d = dft_direct(a, axis=1, inverse=inv)
        assert np.abs(f - d).max() <= 1e-13 * max(1.0, np.abs(d).max())
    assert np.abs(fft_radix2(fft_radix2(a, axis=1), axis=1, inverse=True) - a).max() <= 1e-14 * P
    # cross-check against a library FFT (test only; the oracle never calls it)
    assert np.abs(fft_radix2(a, axis=1) - np.fft.fft(a, axis=1)).max() <= 1e-13 * max(1.0, np.abs(a).sum())


def test_radix2_fft_closed_forms():
    """Delta -> all ones; a single exponential exp(2 pi i k0 n / P) -> P at k0;
    a 3-D separable product transforms to the product of the 1-D transforms."""
    from oracle.fft import fft_radix2, fftn_radix2
    P = 256
    d = np.zeros(P, complex)
    d[0] = 1
    assert np.abs(fft_radix2(d) - 1).max() <= 1e-15
    k0 = 37
    e = np.exp(2j * np.pi * k0 * np.arange(P) / P)
    F = fft_radix2(e)
    ref = np.zeros(P, complex)
    ref[k0] = P
    assert np.abs(F - ref).max() <= 1e-11
    rng = np.random.default_rng(9)
    u, v, w = (rng.standard_normal(n) + 1j * rng.standard_normal(n) for n in (8, 16, 4))
    A = np.einsum("i,j,k->ijk", u, v, w)
    B = np.einsum("i,j,k->ijk", fft_radix2(u), fft_radix2(v), fft_radix2(w))
    assert np.abs(fftn_radix2(A) - B).max() <= 1e-12 * np.abs(B).max()
    with pytest.raises(ValueError):
        fft_radix2(np.ones(12))


def test_oracle_convolution_uses_own_fft():
    """oracle/aim.py performs no library FFT in its arithmetic."""
    import inspect
    import oracle.aim as A
    src = inspect.getsource(A)
    assert "np.fft" not in src and "numpy.fft" not in src and "scipy.fft" not in src


# ------------------------------ the row-sampled checker used by the full-size tests
@pytest.mark.parametrize("name", ["c1", "t_m3", "t_vol", "t_dissim"])
@pytest.mark.parametrize("R", [1, 3])
def test_matvec_rows_equals_full_matvec(name, R):
    """OraclePlan.matvec_rows (far field by the FFT path, interpolation and
    near rows restricted to `rows`) is the reference of every full-size GPU
    parity test: it must equal the rows of the full product, computed through
    the sparse P^T interpolation and the full near matrix.  (t_dissim: its
    full near matrix takes minutes to build, so there the near rows are
    checked against the rows of a larger row set that contains them, and the
    far rows against the full far field.)"""
    P = oracle_plan(name)
    x = make_vectors(P.N, R, 4)
    rng = np.random.default_rng(R)
    rows = np.unique(np.concatenate([[0, P.N - 1], rng.integers(0, P.N, 40)]))
    part = P.matvec_rows(x, rows, method="fft")
    Phi = P.convolve_fft(P.project(x))
    far_full = P.interpolate(Phi)
    scale = np.abs(part).max()
    assert np.abs(P.interpolate(Phi, rows) - far_full[rows]).max() <= 1e-13 * scale
    assert np.abs(P.far(x, "fft", rows=rows) - far_full[rows]).max() <= 1e-13 * scale
    if name != "t_dissim":
        full = P.matvec(x, method="fft")
        assert np.abs(part - full[rows]).max() <= 1e-13 * np.abs(full).max()
        Zr = P.near_matrix(rows).toarray()
        assert np.abs(Zr - P.near_full()[rows].toarray()).max() <= 1e-15 * np.abs(Zr).max()
    else:
        sup = np.unique(np.concatenate([rows, rng.integers(0, P.N, 60)]))
        pos = np.searchsorted(sup, rows)
        Zr = P.near_matrix(rows).toarray()
        assert np.abs(Zr - P.near_matrix(sup).toarray()[pos]).max() <= 1e-15 * np.abs(Zr).max()
        assert np.abs(part - (far_full[rows] + P.near_matrix(sup)[pos] @ x)).max() <= 1e-13 * scale
    # the direct-sum far field agrees with the FFT far field on the sampled rows
    if P.Ng <= 4000:
        assert np.abs(P.matvec_rows(x, rows, method="direct") - part).max() <= 1e-12 * np.abs(part).max()


@pytest.mark.parametrize("name", ["c1", "t_m3", "t_dissim", "t_vol"])
def test_near_pairs_equal_brute_force(name):
    """D5: the k-d tree candidate search returns exactly the brute-force list
    ||c_m - c_n|| <= r (1 + 1e-9) over all n (near_columns), ties included."""
    P = oracle_plan(name)
    rows = np.unique(np.concatenate([[0, P.N - 1], np.random.default_rng(5).integers(0, P.N, 300)]))
    rp, cols = P.near_pairs(rows)
    for i, m in enumerate(rows):
        assert np.array_equal(cols[rp[i]:rp[i + 1]], P.near_columns(m)), m
    for r in (0.0, 10.0):   # degenerate radii: self pairs only / everything
        Q = OraclePlan(make_mesh("t_one"), 2 * np.pi, 0.1, 2, r)
        rp, cols = Q.near_pairs()
        assert rp[-1] == (Q.N if r == 0 else Q.N ** 2)


def test_matvec_golden_files_are_the_oracles():
    """tests/golden/matvec_c*.npz (tools/make_matvec_goldens.py, oracle only):
    metadata, row coverage (every grid x-plane), and -- on C2 -- a few stored
    rows recomputed live with the oracle's row-sampled product."""
    import json
    import os
    from workloads import get_config, make_mesh, make_vectors
    gold = os.path.join(os.path.dirname(__file__), "golden")
    sizes = {"c2": (115200, 16, 500), "c3": (526068, 1, 1000), "c4": (1843200, 1, 1000), "c5": (1119744, 1, 1000)}
    for name, (N, R, nmin) in sizes.items():
        d = np.load(os.path.join(gold, f"matvec_{name}.npz"))
        meta = json.loads(str(d["meta"]))
        assert (meta["N"], meta["nrhs"], meta["x_seed"]) == (N, R, 0)
        assert meta["writer"].startswith("tools/make_matvec_goldens.py")
        assert meta["x_planes_covered"] == meta["x_planes"]
        rows, ref = d["rows"], d["ref"]
        assert rows.size >= nmin and ref.shape == (rows.size, R) and np.all(np.diff(rows) > 0)
        assert rows[0] == 0 and rows[-1] == N - 1 and np.isfinite(ref.view(np.float64)).all()
    cfg = get_config("c2")
    O = OraclePlan(make_mesh(cfg), cfg.k, cfg.h, cfg.M, cfg.near_radius)
    d = np.load(os.path.join(gold, "matvec_c2.npz"))
    pick = np.linspace(0, d["rows"].size - 1, 5).astype(np.int64)
    x = make_vectors(O.N, 16, 0)[:, 5:6].copy()          # one of the 16 columns (they are independent)
    live = O.matvec_rows(x, d["rows"][pick])
    assert np.abs(live - d["ref"][pick][:, 5:6]).max() <= 1e-12 * np.abs(d["ref"]).max()
