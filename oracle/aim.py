"""AIM operator, step by step (§V; readings SURVEY.md §8(c)).

    Z_eq = Z_corr + j k eta0 ( sum_{psi=x,y,z} P_psi^T H P_psi - k^-2 P_phi^T H P_phi )

  * grid: lattice h Z^3 anchored at the world origin (D4); each RWG n is
    assigned the stencil of (M+1)^3 nodes starting at
        s_n = floor(c_n/h - (M-1)/2 + 1e-7)   per axis            (D3)
    ("Each basis function is assigned to a stencil ... N_O + 1 grid points
    in each direction");
  * projection P_psi (step (i)), tensor-moment matching
    (D2): w^psi_{n,(i,j,k)} = sum_q w_q f^psi_n(r_q) L_i(tx) L_j(ty) L_k(tz),
    t = r_q/h - s_n, L the 1-D Lagrange polynomials on nodes 0..M,
    f^{x,y,z} = Lambda_n components, f^phi = div Lambda_n;
  * convolution H (step (ii), eq. AIM_step2):
    H_uv = G(h |u - v|) with G(0) = 0 (D6); by direct summation or by a
    zero-padded FFT with the min-image kernel (D11, D12);
  * interpolation I_psi = P_psi^T (Galerkin, step (iii));
  * near list: ||c_m - c_n|| <= r (1 + 1e-9)  (D5; PAPER.md:527 uses
    N_NF stencils, BASELINE.json a Euclidean radius);
  * precorrection ("computed by eq. Gouter1 with some
    pre-correction"): Z_corr = Z_ex_sym - Z_grid on near pairs, with
    Z_grid = j k eta0 [sum_xyz w_m^T H w_n - k^-2 w_m^phi^T H w_n^phi].

Node order inside a stencil: u = (i (M+1) + j)(M+1) + k (z fastest).
Grid node linear index: (x Ny + y) Nz + z relative to the grid origin.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .constants import ETA0
from .efie import EfieContext, efie_entries_sym
from .fft import fftn_radix2
from .green import green_grid


# ----------------------------------------------------------------- stencils
def stencil_bases(centres, h, M):
    """D3: s = floor(c/h - (M-1)/2 + 1e-7), per axis (int64)."""
    return np.floor(np.asarray(centres) / h - (M - 1) / 2.0 + 1e-7).astype(np.int64)


def grid_box(bases, M):
    """D4: bounding box of all stencil nodes -> (origin int3, dims int3)."""
    origin = bases.min(axis=0)
    dims = bases.max(axis=0) + M + 1 - origin
    return origin, dims


def lagrange(tau, M):
    """1-D Lagrange basis on nodes 0..M:  L_i(t) = prod_{j != i} (t - j)/(i - j)."""
    tau = np.asarray(tau, dtype=np.float64)
    out = np.ones(tau.shape + (M + 1,))
    for i in range(M + 1):
        for j in range(M + 1):
            if j != i:
                out[..., i] *= (tau - j) / (i - j)
    return out


def stencil_offsets(M):
    """(S,3) integer offsets (i,j,k) in stencil order u = (i(M+1)+j)(M+1)+k."""
    r = np.arange(M + 1)
    i, j, k = np.meshgrid(r, r, r, indexing="ij")
    return np.stack([i.ravel(), j.ravel(), k.ravel()], axis=1)


def projection_weights(ctx: EfieContext, bases, h, M, rows=None, chunk=4096):
    """W[n][u][c], c in (x, y, z, phi)  (D2).  rows: optional subset of RWGs."""
    rows = np.arange(ctx.rwg.shape[0]) if rows is None else np.asarray(rows)
    S = (M + 1) ** 3
    W = np.zeros((rows.size, S, 4))
    for s0 in range(0, rows.size, chunk):
        nn = rows[s0:s0 + chunk]
        acc = np.zeros((nn.size, M + 1, M + 1, M + 1, 4))
        for side in (0, 1):
            t = ctx.side_tri[nn, side]
            a = ctx.side_alpha[nn, side]
            p = ctx.side_p[nn, side]
            rq = ctx.qpts[t]                 # (c,7,3)
            wq = ctx.qw[t]                   # (c,7)
            f = np.empty(rq.shape[:2] + (4,))
            f[..., :3] = a[:, None, None] * (rq - p[:, None, :])
            f[..., 3] = 2.0 * a[:, None]
            tau = rq / h - bases[nn][:, None, :]
            Lx = lagrange(tau[..., 0], M)
            Ly = lagrange(tau[..., 1], M)
            Lz = lagrange(tau[..., 2], M)
            acc += np.einsum("cq,cqi,cqj,cqk,cqd->cijkd", wq, Lx, Ly, Lz, f)
        W[s0:s0 + nn.size] = acc.reshape(nn.size, S, 4)
    return W


# ------------------------------------------------------------------ plan
class OraclePlan:
    """All oracle-side operator data for one mesh and AIM parameter set."""

    def __init__(self, mesh, k, h, M, near_radius):
        self.ctx = EfieContext(mesh.vertices, mesh.triangles, mesh.rwg, k)
        self.k, self.h, self.M, self.r = float(k), float(h), int(M), float(near_radius)
        self.N = mesh.rwg.shape[0]
        self.centres = self.ctx.geo["centre"]
        self.bases = stencil_bases(self.centres, h, M)
        self.origin, self.dims = grid_box(self.bases, M)
        self.S = (M + 1) ** 3
        self.offsets = stencil_offsets(M)
        self.W = projection_weights(self.ctx, self.bases, h, M)
        self._P = None
        self._near = None

    # node indices of every RWG's stencil, (N,S) int64
    def stencil_nodes(self, rows=None):
        b = self.bases if rows is None else self.bases[rows]
        g = b[:, None, :] + self.offsets[None, :, :] - self.origin
        Nx, Ny, Nz = self.dims
        return (g[..., 0] * Ny + g[..., 1]) * Nz + g[..., 2]

    @property
    def Ng(self):
        return int(np.prod(self.dims))

    def projection_matrices(self):
        """P_c (Ng x N) sparse, c = x, y, z, phi (step (i))."""
        if self._P is None:
            nodes = self.stencil_nodes()
            cols = np.repeat(np.arange(self.N), self.S)
            self._P = [sp.csr_matrix((self.W[:, :, c].ravel(), (nodes.ravel(), cols)),
                                     shape=(self.Ng, self.N)) for c in range(4)]
        return self._P

    # -------------------------------------------------------------- stages
    def project(self, x):
        """Q_c = P_c x, returned as (4, Nx, Ny, Nz, R)."""
        x = _as2d(x)
        P = self.projection_matrices()
        Q = np.stack([P[c] @ x for c in range(4)])
        return Q.reshape((4,) + tuple(self.dims) + (x.shape[1],))

    def kernel_matrix(self):
        """Dense H (Ng x Ng), H_uv = G(h|u-v|), G(0)=0 -- tiny grids only."""
        Nx, Ny, Nz = self.dims
        g = np.stack(np.meshgrid(np.arange(Nx), np.arange(Ny), np.arange(Nz), indexing="ij"), -1).reshape(-1, 3)
        d = np.linalg.norm((g[:, None, :] - g[None, :, :]).astype(np.float64), axis=2)
        return green_grid(self.h * d, self.k)

    def convolve_direct(self, Q):
        """Phi = H Q by direct O(Ng^2) summation (plain definition)."""
        H = self.kernel_matrix()
        sh = Q.shape
        Qf = Q.reshape(4, self.Ng, sh[-1])
        return np.stack([H @ Qf[c] for c in range(4)]).reshape(sh)

    def convolve_fft(self, Q, pads=None):
        """Phi = H Q by zero-padded FFT with the min-image kernel (D11, D12),
        on power-of-two padded sizes with the oracle's own radix-2 FFT
        (oracle/fft.py; north_star "its own radix-2 FFT")."""
        dims = tuple(int(d) for d in self.dims)
        if pads is None:
            pads = tuple(int(2 ** np.ceil(np.log2(2 * d - 1))) if d > 1 else 1 for d in dims)
        K = self.kernel_samples(pads)
        Kh = fftn_radix2(K)
        out = np.empty_like(Q)
        for c in range(Q.shape[0]):
            for r in range(Q.shape[-1]):
                q = np.zeros(pads, dtype=np.complex128)
                q[: dims[0], : dims[1], : dims[2]] = Q[c, ..., r]
                phi = fftn_radix2(fftn_radix2(q) * Kh, inverse=True)
                out[c, ..., r] = phi[: dims[0], : dims[1], : dims[2]]
        return out

    def kernel_samples(self, pads):
        ax = [np.minimum(np.arange(P), P - np.arange(P)) for P in pads]
        i, j, k = np.meshgrid(*ax, indexing="ij")
        R = self.h * np.sqrt((i * i + j * j + k * k).astype(np.float64))
        return green_grid(R, self.k)

    def interpolate(self, Phi, rows=None):
        """y_far = j k eta0 [sum_xyz P_c^T Phi_c - k^-2 P_phi^T Phi_phi] (step (iii))."""
        R = Phi.shape[-1]
        Pf = Phi.reshape(4, self.Ng, R)
        if rows is None:
            P = self.projection_matrices()
            acc = sum(P[c].T @ Pf[c] for c in range(3)) - (P[3].T @ Pf[3]) / self.k ** 2
        else:
            rows = np.asarray(rows)
            nodes = self.stencil_nodes(rows)                      # (m,S)
            w = self.W[rows]                                      # (m,S,4)
            acc = sum(np.einsum("ms,msr->mr", w[:, :, c], Pf[c][nodes]) for c in range(3))
            acc = acc - np.einsum("ms,msr->mr", w[:, :, 3], Pf[3][nodes]) / self.k ** 2
        return 1j * self.k * ETA0 * acc

    # ---------------------------------------------------------- near field
    def near_columns(self, m):
        """D5: sorted n with ||c_m - c_n|| <= r (1 + 1e-9)."""
        d = np.sqrt(((self.centres - self.centres[m]) ** 2).sum(axis=1))
        return np.nonzero(d <= self.r * (1.0 + 1e-9))[0]

    def near_pairs(self, rows=None, chunk=512):
        """D5 near list of `rows` as CSR (row_ptr, sorted columns).

        Candidates come from a k-d tree ball query (scipy.spatial, a library
        neighbour search used as one step) with a radius 1e-6 larger than
        D5's; each candidate is then kept iff the D5 test on the same
        distance formula as near_columns holds, so the list equals the
        brute-force one (pinned in tests/test_oracle_aim.py)."""
        from scipy.spatial import cKDTree
        rows = np.arange(self.N) if rows is None else np.asarray(rows)
        if getattr(self, "_tree", None) is None:
            self._tree = cKDTree(self.centres)
        rp, cols = [0], []
        lim = self.r * (1.0 + 1e-9)
        for s in range(0, rows.size, chunk):
            rr = rows[s:s + chunk]
            cand = self._tree.query_ball_point(self.centres[rr], self.r * (1.0 + 1e-6) + 1e-12)
            for i in range(rr.size):
                c = np.sort(np.asarray(cand[i], dtype=np.int64))
                d = np.sqrt(((self.centres[c] - self.centres[rr[i]]) ** 2).sum(axis=1))
                c = c[d <= lim]
                cols.append(c)
                rp.append(rp[-1] + c.size)
        return np.asarray(rp), (np.concatenate(cols) if cols else np.zeros(0, np.int64))

    def grid_entries(self, m, n):
        """Z_grid[m,n] = j k eta0 [sum_xyz w_m^T H w_n - k^-2 w_m^phi^T H w_n^phi].

        H_{S_m,S_n}[u,v] = G(h |(s_m + o_u) - (s_n + o_v)|), G(0) = 0.  The
        block depends only on s_m - s_n, so pairs are grouped by it and each
        block is formed once."""
        m = np.asarray(m, dtype=np.int64)
        n = np.asarray(n, dtype=np.int64)
        out = np.zeros(m.size, dtype=np.complex128)
        if m.size == 0:
            return out
        ds = self.bases[m] - self.bases[n]
        keys, inv = np.unique(ds, axis=0, return_inverse=True)
        inv = inv.ravel()
        order = np.argsort(inv, kind="stable")
        bounds = np.searchsorted(inv[order], np.arange(keys.shape[0] + 1))
        o = self.offsets
        for g in range(keys.shape[0]):
            sel = order[bounds[g]:bounds[g + 1]]
            dlt = keys[g][None, None, :] + o[:, None, :] - o[None, :, :]        # (S,S,3)
            H = green_grid(self.h * np.sqrt((dlt.astype(np.float64) ** 2).sum(axis=2)), self.k)
            Wn = self.W[n[sel]]                                                  # (c,S,4)
            T = np.einsum("uv,cvd->cud", H, Wn)                                  # H w_n
            prod = (self.W[m[sel]] * T).sum(axis=1)                              # (c,4)
            out[sel] = 1j * self.k * ETA0 * (prod[:, :3].sum(axis=1) - prod[:, 3] / self.k ** 2)
        return out

    def exact_entries(self, m, n):
        return efie_entries_sym(self.ctx, m, n)

    def near_matrix(self, rows=None):
        """Precorrected near rows as CSR (rows x N): Z_ex_sym - Z_grid."""
        rows_arr = np.arange(self.N) if rows is None else np.asarray(rows)
        rp, cols = self.near_pairs(rows_arr)
        mm = np.repeat(rows_arr, np.diff(rp))
        vals = self.exact_entries(mm, cols) - self.grid_entries(mm, cols)
        return sp.csr_matrix((vals, cols, rp), shape=(rows_arr.size, self.N))

    def near_full(self):
        if self._near is None:
            self._near = self.near_matrix()
        return self._near

    # ------------------------------------------------------------- matvec
    def far(self, x, method="auto", rows=None):
        Q = self.project(x)
        if method == "auto":
            method = "direct" if self.Ng <= 4000 else "fft"
        Phi = self.convolve_direct(Q) if method == "direct" else self.convolve_fft(Q)
        return self.interpolate(Phi, rows)

    def matvec(self, x, method="auto"):
        """y = Z_eq x (all rows)."""
        x2 = _as2d(x)
        y = self.far(x2, method) + self.near_full() @ x2
        return y if np.ndim(x) == 2 else y[:, 0]

    def matvec_rows(self, x, rows, method="auto"):
        """y[rows] = (Z_eq x)[rows] without building the full near matrix."""
        x2 = _as2d(x)
        y = self.far(x2, method, rows=rows) + self.near_matrix(rows) @ x2
        return y if np.ndim(x) == 2 else y[:, 0]


def _as2d(x):
    x = np.asarray(x, dtype=np.complex128)
    return x[:, None] if x.ndim == 1 else x
