"""Free-space Green's function:

    G(r, r') = exp(-j k0 |r - r'|) / (4 pi |r - r'|)      (e^{+j omega t})

green_grid:   the sampled kernel of the AIM convolution H, with G(0) = 0 (D6,
              SPEC.md:457).
green_smooth: G_s(R) = G(R) - 1/(4 pi R) = (exp(-jkR) - 1)/(4 pi R), the
              regular remainder used by singularity subtraction (D8); written
              as (-2 sin^2(kR/2) - j sin kR)/(4 pi R), with G_s(0) = -jk/(4 pi).
"""
from __future__ import annotations

import numpy as np


def green(R, k):
    R = np.asarray(R, dtype=np.float64)
    return np.exp(-1j * k * R) / (4.0 * np.pi * R)


def green_grid(R, k):
    """G(R) with the self term G(0) set to 0 (D6)."""
    R = np.asarray(R, dtype=np.float64)
    out = np.zeros(R.shape, dtype=np.complex128)
    nz = R > 0
    out[nz] = green(R[nz], k)
    return out


def green_smooth(R, k):
    R = np.asarray(R, dtype=np.float64)
    out = np.empty(R.shape, dtype=np.complex128)
    nz = R > 0
    Rn = R[nz]
    out[nz] = (-2.0 * np.sin(0.5 * k * Rn) ** 2 - 1j * np.sin(k * Rn)) / (4.0 * np.pi * Rn)
    out[~nz] = -1j * k / (4.0 * np.pi)
    return out
