"""Block-Jacobi preconditioner over the array elements (SURVEY.md §8(f)
NEXT-4; reading D18 in DESIGN.md).  TEST INFRASTRUCTURE ONLY.

The paper solves its systems "iteratively using GMRES with an ILU-2
preconditioner" (§VI-A); SPEC.md:493-501 substitutes a
per-element block method ("applies per-element dense LU solves of the
diagonal blocks").  Reading D18:

  * elements = connected surfaces of the mesh (triangles joined by an RWG);
    element order = order of their smallest RWG id; RWGs of an element in
    ascending id;
  * block of element e: M_e = Z_ex_sym[e, e] over ALL RWG pairs of e
    (efie.efie_entries_sym: exact symmetrised Galerkin entries, D8, D9);
  * elements that are translates of an earlier element (same number of RWGs,
    same local triangle / vertex numbering, triangle corners equal to 1e-9 of
    the element size after removing the translation) use that element's
    block ("only need to be calculated once for each distinct element",
    PAPER.md:422-425);
  * M^-1 applied blockwise with the explicit inverse (numpy.linalg.inv, a
    library step); right preconditioning Z M^-1 u = V, J = M^-1 u.
"""
from __future__ import annotations

import numpy as np

from .efie import EfieContext, efie_entries_sym


def elements(rwg, n_tri):
    """Connected surfaces: list of ascending RWG-id arrays, ordered by smallest id."""
    rwg = np.asarray(rwg)
    parent = list(range(n_tri))

    def find(a):
        while parent[a] != a:
            parent[a] = parent[parent[a]]
            a = parent[a]
        return a

    for tp, tm in rwg[:, 2:4]:
        a, b = find(int(tp)), find(int(tm))
        if a != b:
            parent[max(a, b)] = min(a, b)
    root_of = {}
    groups = []
    for n in range(rwg.shape[0]):
        r = find(int(rwg[n, 2]))
        if r not in root_of:
            root_of[r] = len(groups)
            groups.append([])
        groups[root_of[r]].append(n)
    return [np.asarray(g, dtype=np.int64) for g in groups]


def _is_translate(ctx: EfieContext, a, b):
    """Element b (RWG ids) a translate of element a (D18 rule)."""
    if a.size != b.size:
        return False
    tri = ctx.triangles
    ta = ctx.side_tri[a]          # (n, 2)
    tb = ctx.side_tri[b]
    if not np.array_equal(ta - ta.min(), tb - tb.min()):
        return False
    va = tri[ta] - tri[ta].min()
    vb = tri[tb] - tri[tb].min()
    if not np.array_equal(va, vb):
        return False
    ca = ctx.vertices[tri[ta]]     # (n, 2, 3, 3) corners
    cb = ctx.vertices[tri[tb]]
    oa = ctx.vertices[tri[ta.min()]][0]
    ob = ctx.vertices[tri[tb.min()]][0]
    da, db = ca - oa, cb - ob
    return bool(np.abs(da - db).max() <= 1e-9 * max(1.0, np.abs(da).max()))


class BlockJacobi:
    """M^-1 for the mesh of `ctx` (D18)."""

    def __init__(self, ctx: EfieContext, build=True):
        self.ctx = ctx
        self.elems = elements(ctx.rwg, ctx.triangles.shape[0])
        self.reps = []          # element index of each distinct block
        self.map = []           # distinct block of each element
        for e, idx in enumerate(self.elems):
            d = next((q for q, r in enumerate(self.reps) if _is_translate(ctx, self.elems[r], idx)), None)
            if d is None:
                d = len(self.reps)
                self.reps.append(e)
            self.map.append(d)
        self.blocks = []
        self.inverses = []
        for r in (self.reps if build else []):
            idx = self.elems[r]
            m, n = np.meshgrid(idx, idx, indexing="ij")
            B = efie_entries_sym(ctx, m.ravel(), n.ravel()).reshape(idx.size, idx.size)
            self.blocks.append(B)
            self.inverses.append(np.linalg.inv(B))

    def apply(self, v):
        """M^-1 v (v: [N] or [N][R])."""
        v = np.asarray(v, dtype=np.complex128)
        out = np.empty_like(v)
        for idx, d in zip(self.elems, self.map):
            out[idx] = self.inverses[d] @ v[idx]
        return out

    def apply_M(self, v):
        """M v (for pins)."""
        v = np.asarray(v, dtype=np.complex128)
        out = np.empty_like(v)
        for idx, d in zip(self.elems, self.map):
            out[idx] = self.blocks[d] @ v[idx]
        return out


def gmres_right(gmres, matvec, precond, b, **kw):
    """Right-preconditioned restarted GMRES: solve (Z M^-1) u = b with the
    oracle's gmres, return J = M^-1 u (the true residual b - Z J equals the
    one gmres tracks, b - (Z M^-1) u)."""
    res = gmres(lambda u: matvec(precond(u)), b, **kw)
    res = dict(res)
    res["x"] = precond(res["x"])
    return res
