"""Seeded synthetic macromodel blocks for the reduced system of
PAPER.md eq. finalsystem, (D - G T A^-1 B) E^ = V^.

The paper's blocks come from each element's scatterer (interior MoM matrix
A_m, coupling B_m, transfer T_m) and the dual-basis Gram
matrix D_m; the scatterer geometries are not available
(DESIGN.md §3, §11), so -- as SURVEY.md §8(f) plans -- the benchmark and the
parity tests use seeded random blocks of the paper's shapes: N_m = ratio x
N^_m interior unknowns (PAPER.md:659, 840, 953 give N_m / N^_m of about 4-10),
D_m diagonally dominant ("D is well-conditioned because it is diagonally
dominant"), A_m well conditioned.  NO method arithmetic here:
only random matrices, drawn with numpy's default_rng in a fixed order.
"""
from __future__ import annotations

import numpy as np

ETA0 = 4e-7 * np.pi * 299792458.0   # scale of B only (so Z K is O(1) next to D)


def _cn(g, shape):
    return (g.standard_normal(shape) + 1j * g.standard_normal(shape)) / np.sqrt(2.0)


def macromodel_blocks(nhat: int, ratio: int = 4, seed: int = 0):
    """(D [nhat][nhat], T [nhat][n], A [n][n], B [n][nhat]) complex128, n = ratio nhat:
    D = I + 0.1 R/sqrt(nhat), T = R/sqrt(n), A = 2 I + R/sqrt(n), B = R/(eta0 sqrt(nhat))."""
    n = ratio * nhat
    g = np.random.default_rng(seed)
    D = np.eye(nhat) + 0.1 * _cn(g, (nhat, nhat)) / np.sqrt(nhat)
    T = _cn(g, (nhat, n)) / np.sqrt(n)
    A = 2.0 * np.eye(n) + _cn(g, (n, n)) / np.sqrt(n)
    B = _cn(g, (n, nhat)) / (ETA0 * np.sqrt(nhat))
    return D, T, A, B


def type_blocks(sizes, ratio: int = 4, seed: int = 0):
    """Blocks of every element type d (size sizes[d]), seeds seed + d."""
    return [macromodel_blocks(int(s), ratio, seed + d) for d, s in enumerate(sizes)]
