"""The oracle's own radix-2 FFT (BASELINE.json north_star: "direct-summation
grid convolution on tiny grids, its own radix-2 FFT beyond that"; SURVEY.md
§8(c) step 5).  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Used by aim.convolve_fft for step (ii) of the AIM matvec, the zero-padded
convolution of eq. AIM_step2, on power-of-two padded
sizes (reading D11: any P >= 2N - 1 gives the same linear convolution).

Definition (numpy's sign convention):

    forward   X[k] = sum_{n=0}^{P-1} x[n] exp(-2 pi i k n / P)
    inverse   x[n] = (1/P) sum_{k=0}^{P-1} X[k] exp(+2 pi i k n / P)

Algorithm: iterative decimation-in-time Cooley-Tukey.  The input is put in
bit-reversed order, then log2(P) butterfly stages combine pairs of
half-length transforms of size m into transforms of size 2m:

    X[k]     = E[k] + w^k O[k]
    X[k + m] = E[k] - w^k O[k],      w = exp(-+ 2 pi i / (2m)),  0 <= k < m.

Plain numpy, vectorised over every other axis; no library FFT is called.
Pinned in tests/test_oracle_aim.py against a direct O(P^2) DFT (P <= 64),
closed forms (delta, single exponential) and the direct-sum convolution.
"""
from __future__ import annotations

import numpy as np


def bit_reverse_permutation(P):
    """idx[n] = n with its log2(P) bits reversed."""
    bits = int(P).bit_length() - 1
    idx = np.zeros(P, dtype=np.int64)
    n = np.arange(P, dtype=np.int64)
    for b in range(bits):
        idx |= ((n >> b) & 1) << (bits - 1 - b)
    return idx


def fft_radix2(a, axis=-1, inverse=False):
    """1-D radix-2 FFT of `a` along `axis` (length must be a power of two)."""
    a = np.moveaxis(np.asarray(a, dtype=np.complex128), axis, -1)
    P = a.shape[-1]
    if P & (P - 1):
        raise ValueError(f"radix-2 FFT needs a power-of-two length, got {P}")
    lead = a.shape[:-1]
    x = a[..., bit_reverse_permutation(P)]          # copy, bit-reversed order
    sign = 1.0 if inverse else -1.0
    m = 1
    while m < P:
        w = np.exp(sign * 2j * np.pi * np.arange(m) / (2 * m))
        x = x.reshape(lead + (P // (2 * m), 2, m))
        e = x[..., 0, :]
        o = x[..., 1, :] * w
        x = np.stack([e + o, e - o], axis=-2).reshape(lead + (P,))
        m *= 2
    if inverse:
        x = x / P
    return np.moveaxis(x, -1, axis)


def fftn_radix2(a, inverse=False):
    """Multi-dimensional transform: the 1-D transform applied along every
    axis -- radix-2 on power-of-two lengths (the oracle's sizes), the direct
    DFT on any other length (only the small padding-independence pins of
    reading D11 use those)."""
    x = np.asarray(a, dtype=np.complex128)
    for ax in range(x.ndim):
        P = x.shape[ax]
        if P & (P - 1) == 0:
            x = fft_radix2(x, axis=ax, inverse=inverse)
        else:
            x = dft_direct(x, axis=ax, inverse=inverse)
    return x


def dft_direct(a, axis=-1, inverse=False):
    """O(P^2) direct DFT (the plain definition), for pinning the FFT."""
    a = np.moveaxis(np.asarray(a, dtype=np.complex128), axis, -1)
    P = a.shape[-1]
    n = np.arange(P)
    sign = 1.0 if inverse else -1.0
    F = np.exp(sign * 2j * np.pi * np.outer(n, n) / P)
    out = a @ F.T
    if inverse:
        out = out / P
    return np.moveaxis(out, -1, axis)
