"""Closed cube-surface meshes and cube arrays.

The "equivalent surfaces" of the paper (§II-A) are, in the
BASELINE.json configs, closed cube surfaces with no scatterer inside.  Each
face is split into n x n squares and each square is cut along the diagonal
(u_i, v_j)-(u_{i+1}, v_{j+1}) in face axes (u, v) = cyclic (y,z), (z,x), (x,y),
with outward winding; vertices are shared within a cube.

RWG table ("RWG basis function"): one RWG per interior edge,
rows sorted by (min vid, max vid); row = {va, vb, t_plus, t_minus} with
t_plus the lower triangle index.
"""
from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np


@dataclass
class Mesh:
    vertices: np.ndarray   # float64 [nv][3]
    triangles: np.ndarray  # int32 [nt][3]
    rwg: np.ndarray        # int32 [N][4] = {va, vb, t_plus, t_minus}

    @property
    def n_rwg(self) -> int:
        return int(self.rwg.shape[0])


# face axes (u, v) for normal axis a, cyclic so that u x v = +a
_FACE_UV = {0: (1, 2), 1: (2, 0), 2: (0, 1)}


@lru_cache(maxsize=None)
def _unit_cube_template(n: int):
    """Integer lattice vertices (in [0,n]^3) and triangles of one cube surface."""
    index = {}
    verts = []
    # surface lattice points in lexicographic (i, j, k) order
    for i in range(n + 1):
        for j in range(n + 1):
            for k in range(n + 1):
                if i in (0, n) or j in (0, n) or k in (0, n):
                    index[(i, j, k)] = len(verts)
                    verts.append((i, j, k))
    tris = []
    for a in range(3):
        u, v = _FACE_UV[a]
        for side in (0, n):
            outward_plus = side == n
            for iu in range(n):
                for iv in range(n):
                    def node(du, dv):
                        p = [0, 0, 0]
                        p[a] = side
                        p[u] = iu + du
                        p[v] = iv + dv
                        return index[tuple(p)]
                    c00, c10, c11, c01 = node(0, 0), node(1, 0), node(1, 1), node(0, 1)
                    if outward_plus:
                        tris.append((c00, c10, c11))
                        tris.append((c00, c11, c01))
                    else:
                        tris.append((c00, c11, c10))
                        tris.append((c00, c01, c11))
    verts = np.asarray(verts, dtype=np.float64)
    tris = np.asarray(tris, dtype=np.int64)
    rwg = rwg_edges_from_triangles(tris)
    return verts, tris, rwg


def rwg_edges_from_triangles(tris: np.ndarray) -> np.ndarray:
    """Interior edges of a closed triangle mesh -> RWG rows {va, vb, t+, t-}.

    Raises ValueError if some edge is not shared by exactly two triangles
    (open or non-manifold mesh).
    """
    tris = np.asarray(tris, dtype=np.int64)
    nt = tris.shape[0]
    e = np.concatenate([tris[:, [0, 1]], tris[:, [1, 2]], tris[:, [2, 0]]], axis=0)
    tid = np.concatenate([np.arange(nt)] * 3)
    lo = e.min(axis=1)
    hi = e.max(axis=1)
    order = np.lexsort((tid, hi, lo))
    lo, hi, tid = lo[order], hi[order], tid[order]
    if lo.size % 2:
        raise ValueError("mesh is not closed")
    same = (lo[0::2] == lo[1::2]) & (hi[0::2] == hi[1::2])
    if not same.all():
        raise ValueError("mesh is not closed / not 2-manifold")
    if lo.size > 2:
        # an edge used by more than two triangles
        key = lo[0::2] * (hi.max() + 1) + hi[0::2]
        if np.unique(key).size != key.size:
            raise ValueError("non-manifold edge")
    va, vb = lo[0::2], hi[0::2]
    tp, tm = tid[0::2], tid[1::2]  # lexsort on tid -> t+ is the lower index
    return np.stack([va, vb, tp, tm], axis=1).astype(np.int32)


def cube_surface(center, side: float, n: int) -> Mesh:
    lat, tris, rwg = _unit_cube_template(n)
    c = np.asarray(center, dtype=np.float64)
    verts = c - side / 2.0 + lat * (side / n)
    return Mesh(verts, tris.astype(np.int32), rwg.copy())


def cube_array(centers, sides, ns) -> Mesh:
    """Concatenate cube surfaces element by element (element-blocked ids).

    Because vertex ids are element-blocked and each cube's RWG rows are sorted
    by (min vid, max vid), the concatenation is globally sorted as well.
    """
    vs, ts, rs = [], [], []
    voff = 0
    toff = 0
    for c, s, n in zip(centers, sides, ns):
        lat, tris, rwg = _unit_cube_template(int(n))
        verts = np.asarray(c, dtype=np.float64) - s / 2.0 + lat * (s / n)
        vs.append(verts)
        ts.append(tris + voff)
        r = rwg.astype(np.int64).copy()
        r[:, :2] += voff
        r[:, 2:] += toff
        rs.append(r)
        voff += verts.shape[0]
        toff += tris.shape[0]
    return Mesh(np.concatenate(vs).astype(np.float64),
                np.concatenate(ts).astype(np.int32),
                np.concatenate(rs).astype(np.int32))
