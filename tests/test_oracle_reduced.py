"""Pins of the oracle's reduced-system product (oracle/reduced.py; PAPER.md
eq. finalsystem / MV_product1)."""
import numpy as np

from conftest import oracle_plan
from oracle.precond import elements
from oracle.reduced import ReducedSystem
from workloads import make_vectors
from workloads.macromodel import macromodel_blocks, type_blocks


def test_identity_blocks_reduce_to_one_plus_Z():
    """D = T = A = B = I (N_m = N^_m): (D - G T A^-1 B) Y = Y + Z_eq Y (G = -Z_eq, D1)."""
    P = oracle_plan("c1")
    el = elements(P.ctx.rwg, P.ctx.triangles.shape[0])
    n = el[0].size
    I = np.eye(n, dtype=complex)
    R = ReducedSystem(P, el, [0] * len(el), [(I, I, I, I)])
    Y = make_vectors(P.N, 1, 3)[:, 0]
    assert np.abs(R.matvec(Y) - (Y + P.matvec(Y))).max() <= 1e-12 * np.abs(P.matvec(Y)).max()


def test_block_algebra_and_linearity():
    """K = T A^-1 B applied per element equals the explicit dense product;
    the operator is linear."""
    P = oracle_plan("c1")
    el = elements(P.ctx.rwg, P.ctx.triangles.shape[0])
    blocks = type_blocks([el[0].size], ratio=2, seed=4)
    R = ReducedSystem(P, el, [0] * len(el), blocks)
    Y = make_vectors(P.N, 2, 5)
    D, T, A, B = blocks[0]
    K = T @ np.linalg.inv(A) @ B
    t = R.apply_K(Y[:, 0])
    for idx in el:
        assert np.abs(t[idx] - K @ Y[idx, 0]).max() <= 1e-12 * np.abs(t).max()
    a = R.matvec(2.0 * Y[:, 0] - 1j * Y[:, 1])
    b = 2.0 * R.matvec(Y[:, 0]) - 1j * R.matvec(Y[:, 1])
    assert np.abs(a - b).max() <= 1e-12 * np.abs(a).max()


def test_synthetic_blocks_seeded_and_shaped():
    D, T, A, B = macromodel_blocks(10, ratio=3, seed=1)
    assert D.shape == (10, 10) and T.shape == (10, 30) and A.shape == (30, 30) and B.shape == (30, 10)
    D2 = macromodel_blocks(10, ratio=3, seed=1)[0]
    assert np.array_equal(D, D2)
    assert np.linalg.cond(A) < 10 and np.linalg.cond(D) < 2
