"""Pins of the oracle's block-Jacobi preconditioner (oracle/precond.py,
reading D18; SPEC.md:493-501 examples)."""
import numpy as np
import pytest

from conftest import oracle_plan
from oracle.aim import OraclePlan
from oracle.efie import dense_Z
from oracle.excitation import plane_wave_rhs
from oracle.gmres import gmres
from oracle.precond import BlockJacobi, elements, gmres_right
from workloads import make_mesh, make_vectors


def test_elements_and_grouping():
    """C1: 4 identical cubes -> 4 elements, 1 distinct block; t_dissim: 9
    cubes of drawn sides -> 9 distinct blocks; a cube rotated by 90 degrees
    is not a translate."""
    P = oracle_plan("c1")
    bj = BlockJacobi(P.ctx)
    assert len(bj.elems) == 4 and len(bj.reps) == 1 and bj.map == [0, 0, 0, 0]
    assert sorted(np.concatenate(bj.elems).tolist()) == list(range(P.N))
    m = make_mesh("t_dissim")
    assert len(elements(m.rwg, m.triangles.shape[0])) == 9
    from oracle.efie import EfieContext
    assert len(BlockJacobi(EfieContext(m.vertices, m.triangles, m.rwg, 2 * np.pi), build=False).reps) == 9
    # rotate the second cube of a 2-cube array about z by 90 degrees: not a translate
    from workloads.meshes import cube_array
    mm = cube_array(np.array([[0, 0, 0], [0.6, 0, 0]]), [0.4, 0.4], [3, 3])
    v = mm.vertices.copy()
    half = v.shape[0] // 2
    c = np.array([0.6, 0, 0])
    r = v[half:] - c
    v[half:] = c + np.stack([-r[:, 1], r[:, 0], r[:, 2]], axis=1)
    ctx = EfieContext(v, mm.triangles, mm.rwg, 2 * np.pi)
    assert len(BlockJacobi(ctx, build=False).reps) == 2
    ctx0 = EfieContext(mm.vertices, mm.triangles, mm.rwg, 2 * np.pi)
    assert len(BlockJacobi(ctx0, build=False).reps) == 1


def test_blocks_equal_dense_matrix_blocks():
    """Each element block equals the element's diagonal block of the dense
    symmetrised exact matrix (efie.dense_Z: every triangle pair, no reuse),
    also for the elements that reuse the first element's block."""
    P = oracle_plan("c1")
    bj = BlockJacobi(P.ctx)
    Zd = dense_Z(P.ctx)
    for idx, d in zip(bj.elems, bj.map):
        B = Zd[np.ix_(idx, idx)]
        assert np.abs(bj.blocks[d] - B).max() <= 1e-9 * np.abs(B).max()


def test_apply_is_block_inverse_and_linear():
    P = oracle_plan("t_vol")
    bj = BlockJacobi(P.ctx)
    x = make_vectors(P.N, 2, 3)
    y = bj.apply(x)
    assert np.abs(bj.apply_M(y) - x).max() <= 1e-9 * np.abs(x).max()
    z = bj.apply(2.0 * x[:, 0] - 1j * x[:, 1])
    assert np.abs(z - (2.0 * y[:, 0] - 1j * y[:, 1])).max() <= 1e-12 * np.abs(z).max()


def test_single_element_all_near_converges_in_one_iteration():
    """1-element problem, exact block inverse -> preconditioned
    GMRES converges in 1 iteration.  With the near radius covering every pair
    the AIM operator equals Z_ex_sym exactly (precorrection), so M = Z_eq."""
    m = make_mesh("t_one")
    P = OraclePlan(m, 2 * np.pi, 0.1, 2, 10.0)
    bj = BlockJacobi(P.ctx)
    V = plane_wave_rhs(P.ctx)
    res = gmres_right(gmres, P.matvec, bj.apply, V, restart=50, tol=1e-10)
    assert res["iters"] == 1 and res["rel_res"] <= 1e-10


def test_preconditioned_gmres_c1():
    """Fewer iterations than unpreconditioned GMRES and the
    true residual of J = M^-1 u below tol."""
    P = oracle_plan("c1")
    bj = BlockJacobi(P.ctx)
    V = plane_wave_rhs(P.ctx)
    r0 = gmres(P.matvec, V, restart=50, tol=1e-4)
    r1 = gmres_right(gmres, P.matvec, bj.apply, V, restart=50, tol=1e-4)
    assert r1["converged"] and r1["iters"] < r0["iters"] / 5
    assert np.linalg.norm(V - P.matvec(r1["x"])) / np.linalg.norm(V) <= 1e-4 * (1 + 1e-6)
