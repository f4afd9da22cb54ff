"""Seeded random sketch and stratified row samples for the full-size parity
tests (test infrastructure; NO method arithmetic).

A Gaussian sketch S v = [<g_i, v>]_{i<k} with g_i ~ CN(0, 1) iid estimates the
L2 norm of a long vector (E|<g,v>|^2 = ||v||^2), so the relative L2 distance
of two solution vectors of 10^6 entries can be checked against a stored
k-entry sketch of the reference (Johnson-Lindenstrauss).  Both the golden
writer (tools/make_goldens.py, oracle only) and the GPU tests draw the same
g_i from numpy's default_rng(seed), in chunks, in a fixed order.
"""
from __future__ import annotations

import numpy as np


def sketch(v, k=32, seed=12345, chunk=1 << 18):
    """[k] complex128: sum_n g_i[n] v[n], g_i[n] = (a + 1j b)/sqrt(2), a, b ~ N(0,1),
    drawn in row-chunks of `chunk` entries (chunk-major, then i, then re/im)."""
    v = np.asarray(v, dtype=np.complex128).ravel()
    out = np.zeros(k, dtype=np.complex128)
    rng = np.random.default_rng(seed)
    for s in range(0, v.size, chunk):
        seg = v[s:s + chunk]
        g = rng.standard_normal((k, 2, seg.size))
        out += ((g[:, 0] + 1j * g[:, 1]) / np.sqrt(2.0)) @ seg
    return out


def stratified_rows(bases, n_random=512, seed=0, slab_bounds=None, tie_mask=None, per_class=32):
    """Row sample for the full-size matvec checks: one RWG per grid x-plane
    (by stencil base x), the first and last RWG, `n_random` uniform rows,
    `per_class` rows of each stencil tie class (tie_mask [N][3] bool: the
    centre coordinate lies on a D3 tie), and two RWGs on either side of every
    slab boundary (base x == X[r] - 1 and X[r]).  Sorted, unique."""
    bases = np.asarray(bases)
    N = bases.shape[0]
    rng = np.random.default_rng(seed)
    bx = bases[:, 0]
    order = np.argsort(bx, kind="stable")
    planes, first = np.unique(bx[order], return_index=True)
    picks = [order[first], [0, N - 1], rng.integers(0, N, n_random)]
    if tie_mask is not None:
        tm = np.asarray(tie_mask, dtype=bool)
        for cls in range(tm.shape[1]):
            idx = np.nonzero(tm[:, cls])[0]
            if idx.size:
                picks.append(rng.choice(idx, min(per_class, idx.size), replace=False))
    if slab_bounds is not None:
        for X in slab_bounds:
            for xb in (X - 1, X):
                idx = np.nonzero(bx - bx.min() == xb)[0]
                if idx.size:
                    picks.append(rng.choice(idx, min(2, idx.size), replace=False))
    return np.unique(np.concatenate([np.asarray(p, dtype=np.int64).ravel() for p in picks]))
