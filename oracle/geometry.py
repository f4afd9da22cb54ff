"""Triangle / RWG geometry and the 7-point quadrature rule.

RWG basis ("the n-th RWG basis function"; orientation as in
SURVEY.md §8(b)):  current flows from t+ across the edge into t-,
    Lambda_n(r) = l/(2A+) (r - p+)   on t+,
    Lambda_n(r) = l/(2A-) (p- - r)   on t-,
    div Lambda_n = +l/A+ on t+,  -l/A- on t-.
Written per triangle t of RWG n as Lambda_n = alpha (r - p_t) with
alpha = sigma l / (2 A_t), sigma = +1 on t+, -1 on t-, div = 2 alpha.

Quadrature (D7): the 7-point degree-5 rule of Radon (Dunavant's 7-point
rule), barycentrics (1/3,1/3,1/3) weight 9/40; (a,a,1-2a) with
a = (6 -+ sqrt15)/21, weights (155 -+ sqrt15)/1200; weights multiply area.
"""
from __future__ import annotations

import math

import numpy as np


class MeshError(ValueError):
    pass


def dunavant7():
    """Barycentric coordinates (7,3) and weights (7,) summing to 1."""
    s15 = math.sqrt(15.0)
    a1 = (6.0 - s15) / 21.0
    a2 = (6.0 + s15) / 21.0
    w1 = (155.0 - s15) / 1200.0
    w2 = (155.0 + s15) / 1200.0
    bary = [(1.0 / 3.0, 1.0 / 3.0, 1.0 / 3.0)]
    wts = [9.0 / 40.0]
    for a, w in ((a1, w1), (a2, w2)):
        b = 1.0 - 2.0 * a
        bary += [(b, a, a), (a, b, a), (a, a, b)]
        wts += [w, w, w]
    return np.array(bary), np.array(wts)


def triangle_geometry(vertices, triangles):
    v = np.asarray(vertices, dtype=np.float64)
    t = np.asarray(triangles, dtype=np.int64)
    p0, p1, p2 = v[t[:, 0]], v[t[:, 1]], v[t[:, 2]]
    cr = np.cross(p1 - p0, p2 - p0)
    twice_area = np.linalg.norm(cr, axis=1)
    area = 0.5 * twice_area
    with np.errstate(invalid="ignore", divide="ignore"):
        normal = cr / twice_area[:, None]
    centroid = (p0 + p1 + p2) / 3.0
    return dict(area=area, normal=normal, centroid=centroid, corners=np.stack([p0, p1, p2], axis=1))


def triangle_quadrature(vertices, triangles):
    """Quadrature points (nt,7,3) and area-scaled weights (nt,7)."""
    g = triangle_geometry(vertices, triangles)
    bary, w = dunavant7()
    pts = np.einsum("qk,tkd->tqd", bary, g["corners"])
    wts = w[None, :] * g["area"][:, None]
    return pts, wts


def validate_mesh(vertices, triangles, rwg):
    """both triangles contain va, vb; t+ != t-; area > 0."""
    v = np.asarray(vertices)
    t = np.asarray(triangles, dtype=np.int64)
    r = np.asarray(rwg, dtype=np.int64)
    if v.ndim != 2 or v.shape[1] != 3 or t.ndim != 2 or t.shape[1] != 3 or r.ndim != 2 or r.shape[1] != 4:
        raise MeshError("bad array shapes")
    if t.size and (t.min() < 0 or t.max() >= v.shape[0]):
        raise MeshError("triangle vertex index out of range")
    if r.size and (r[:, 2:].min() < 0 or r[:, 2:].max() >= t.shape[0]):
        raise MeshError("rwg triangle index out of range")
    area = triangle_geometry(v, t)["area"]
    if np.any(~(area > 0)):
        raise MeshError("degenerate triangle")
    if np.any(r[:, 2] == r[:, 3]):
        raise MeshError("t+ == t-")
    for col in (2, 3):
        tt = t[r[:, col]]
        has_a = (tt == r[:, 0:1]).any(axis=1)
        has_b = (tt == r[:, 1:2]).any(axis=1)
        if not (has_a & has_b).all():
            raise MeshError("rwg edge not contained in its triangle")
    if np.any(r[:, 0] == r[:, 1]):
        raise MeshError("zero-length rwg edge")


def free_vertex(triangles, tri_idx, va, vb):
    """Index of the vertex of triangle tri_idx not on edge (va, vb)."""
    tt = np.asarray(triangles, dtype=np.int64)[tri_idx]
    mask = (tt != va[:, None]) & (tt != vb[:, None])
    return tt[np.arange(tt.shape[0]), mask.argmax(axis=1)]


def rwg_geometry(vertices, triangles, rwg):
    """Per-RWG: edge length l, areas A+/A-, free vertices p+/p-, centre c.

    Centre c_n = 1/2 (centroid(t+) + centroid(t-))  (D3).
    """
    v = np.asarray(vertices, dtype=np.float64)
    r = np.asarray(rwg, dtype=np.int64)
    tg = triangle_geometry(v, triangles)
    va, vb, tp, tm = r[:, 0], r[:, 1], r[:, 2], r[:, 3]
    l = np.linalg.norm(v[vb] - v[va], axis=1)
    fp = free_vertex(triangles, tp, va, vb)
    fm = free_vertex(triangles, tm, va, vb)
    centre = 0.5 * (tg["centroid"][tp] + tg["centroid"][tm])
    return dict(l=l, tp=tp, tm=tm, Ap=tg["area"][tp], Am=tg["area"][tm],
                pp=v[fp], pm=v[fm], centre=centre, va=va, vb=vb)
