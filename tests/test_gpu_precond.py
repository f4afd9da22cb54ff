"""GPU parity of the block-Jacobi preconditioner (SURVEY.md §8(f) NEXT-4,
reading D18) and of the preconditioned / unpreconditioned GMRES (D15)
against the oracle (oracle/precond.py, oracle/gmres.py)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from conftest import oracle_plan  # noqa: E402
from workloads import get_config, make_mesh, make_vectors  # noqa: E402

_BJ = {}


def oracle_bj(name):
    from oracle.precond import BlockJacobi
    if name not in _BJ:
        _BJ[name] = BlockJacobi(oracle_plan(name).ctx)
    return _BJ[name]


def gpu_plan(name, **over):
    from paper_1712_02443_b200 import AimPlan
    cfg = get_config(name)
    p = dict(k=cfg.k, h=cfg.h, M=cfg.M, near_radius=cfg.near_radius)
    p.update(over)
    return AimPlan.from_mesh(make_mesh(cfg), p["k"], p["h"], p["M"], p["near_radius"])


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b))


@pytest.mark.parametrize("name,elems,distinct", [("c1", 4, 1), ("t_vol", 8, 1), ("t_dissim", 9, 9), ("t_m3", 6, 1)])
def test_precond_structure_and_apply(name, elems, distinct):
    """Element grouping equals the oracle's; M^-1 x equals the oracle's
    blockwise numpy inverse to 1e-10 (GEMM path: t_vol, 8 elements share one
    inverse; GEMV path: c1, t_m3, t_dissim)."""
    bj = oracle_bj(name)
    assert len(bj.elems) == elems and len(bj.reps) == distinct
    G = gpu_plan(name)
    info = G.precond_build(1)
    assert info["built"] == 1 and info["elements"] == elems and info["distinct"] == distinct
    assert info["max_block"] == max(e.size for e in bj.elems)
    x = make_vectors(G.N, 1, 9)[:, 0]
    y = G.precond_apply(torch.from_numpy(x).cuda()).cpu().numpy()
    assert rel(y, bj.apply(x)) <= 1e-10
    G.close()


def test_precond_single_element_one_iteration():
    """one element with every pair near (Z_eq = Z_ex_sym = M):
    preconditioned GMRES converges in one iteration."""
    from paper_1712_02443_b200 import AimPlan
    m = make_mesh("t_one")
    G = AimPlan(m.vertices, m.triangles, m.rwg, 2 * np.pi, 0.1, 2, 10.0)
    G.precond_build(1)
    V = G.planewave_rhs()
    J, it, rr, st = G.gmres(V, restart=50, tol=1e-10)
    assert st == "AIM_OK" and it == 1 and rr <= 1e-10
    G.close()


@pytest.mark.parametrize("name", ["c1", "t_vol", "t_dissim"])
def test_preconditioned_gmres_parity(name):
    """D15 with right preconditioning: converged counts within +-1 of the
    oracle's, J at the oracle's count <= 1e-5, residual history <= 1e-6,
    true residual of the GPU's J checked with an oracle matvec; far fewer
    iterations than without the preconditioner."""
    from oracle.excitation import plane_wave_rhs
    from oracle.gmres import gmres
    from oracle.precond import gmres_right
    O = oracle_plan(name)
    bj = oracle_bj(name)
    V = plane_wave_rhs(O.ctx)
    ref = gmres_right(gmres, O.matvec, bj.apply, V, restart=50, tol=1e-4)
    G = gpu_plan(name)
    G.precond_build(1)
    Vt = torch.from_numpy(V).cuda()
    J, it, rr, st = G.gmres(Vt, restart=50, tol=1e-4)
    assert st == "AIM_OK" and abs(it - ref["iters"]) <= 1
    Jn = J.cpu().numpy()
    assert np.linalg.norm(V - O.matvec(Jn)) / np.linalg.norm(V) <= 1e-4 * (1 + 1e-6)
    Jf, itf, rrf, _ = G.gmres(Vt, restart=50, tol=1e-4, fixed_iters=ref["iters"])
    assert itf == ref["iters"]
    assert rel(Jf.cpu().numpy(), ref["x"]) <= 1e-5
    h = G.gmres_history()
    assert h.size == ref["iters"]
    assert np.abs(h - np.asarray(ref["history"])).max() <= 1e-6 * np.abs(ref["history"]).max()
    G.precond_build(0)
    assert G.precond_info()["built"] == 0
    _, it0, _, _ = G.gmres(Vt, restart=50, tol=1e-4)
    assert it0 > 3 * it
    G.close()


def test_gmres_history_and_breakdown_guard():
    """Unpreconditioned history equals the oracle's; a NaN right-hand side
    returns AIM_E_BREAKDOWN instead of iterating on garbage."""
    from oracle.excitation import plane_wave_rhs
    from oracle.gmres import gmres
    from paper_1712_02443_b200 import AimError
    O = oracle_plan("c1")
    V = plane_wave_rhs(O.ctx)
    ref = gmres(O.matvec, V, restart=50, tol=1e-4, fixed_iters=60)
    G = gpu_plan("c1")
    Vt = torch.from_numpy(V).cuda()
    G.gmres(Vt, restart=50, tol=1e-4, fixed_iters=60)
    h = G.gmres_history()
    assert h.size == 60
    assert np.abs(h - np.asarray(ref["history"])).max() <= 1e-6 * np.abs(ref["history"]).max()
    Vb = Vt.clone()
    Vb[5] = complex(float("nan"), 0.0)
    with pytest.raises(AimError) as e:
        G.gmres(Vb, restart=50, tol=1e-4)
    assert e.value.status == -7
    G.close()
