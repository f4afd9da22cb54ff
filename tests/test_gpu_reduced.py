"""GPU parity of the reduced (macromodel) system product and its GMRES
(PAPER.md eq. finalsystem / MV_product1) against the
oracle (oracle/reduced.py) on seeded synthetic macromodel blocks
(workloads/macromodel.py)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from conftest import oracle_plan  # noqa: E402
from workloads import get_config, make_mesh, make_vectors  # noqa: E402
from workloads.macromodel import type_blocks  # noqa: E402


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b))


def setup(name, ratio=2):
    from oracle.precond import BlockJacobi
    from oracle.reduced import ReducedSystem
    from paper_1712_02443_b200 import AimPlan
    cfg = get_config(name)
    O = oracle_plan(name)
    bj = BlockJacobi(O.ctx, build=False)
    G = AimPlan.from_mesh(make_mesh(cfg), cfg.k, cfg.h, cfg.M, cfg.near_radius)
    eo, grp = G.elements()
    # the library enumerates elements and translate groups as the oracle does
    assert grp.tolist() == bj.map
    for e, idx in enumerate(bj.elems):
        assert np.all(eo[idx] == e)
    sizes = [bj.elems[r].size for r in bj.reps]
    blocks = type_blocks(sizes, ratio=ratio, seed=11)
    G.reduced_set(grp, blocks)
    R = ReducedSystem(O, bj.elems, bj.map, blocks)
    return G, R, O


@pytest.mark.parametrize("name", ["c1", "t_vol", "t_dissim"])
def test_reduced_matvec(name):
    """(D - G T A^-1 B) Y <= 1e-10 vs the oracle (GEMM path: t_vol's 8
    elements share a type; GEMV path: c1, t_dissim's 9 types)."""
    G, R, O = setup(name)
    Y = make_vectors(O.N, 1, 6)[:, 0]
    out = G.reduced_matvec(torch.from_numpy(Y).cuda()).cpu().numpy()
    assert rel(out, R.matvec(Y)) <= 1e-10
    G.close()


def test_reduced_gmres_c1():
    """GMRES on the reduced system: converged counts within +-1, E at equal
    counts <= 1e-5, true residual with the oracle's reduced product."""
    from oracle.excitation import plane_wave_rhs
    from oracle.gmres import gmres
    G, R, O = setup("c1")
    V = plane_wave_rhs(O.ctx)
    ref = gmres(R.matvec, V, restart=50, tol=1e-6)
    Vt = torch.from_numpy(V).cuda()
    E, it, rr, st = G.reduced_gmres(Vt, restart=50, tol=1e-6)
    assert st == "AIM_OK" and abs(it - ref["iters"]) <= 1
    En = E.cpu().numpy()
    assert np.linalg.norm(V - R.matvec(En)) / np.linalg.norm(V) <= 1e-6 * (1 + 1e-6)
    Ef, itf, _, _ = G.reduced_gmres(Vt, restart=50, tol=1e-6, fixed_iters=ref["iters"])
    assert itf == ref["iters"] and rel(Ef.cpu().numpy(), ref["x"]) <= 1e-5
    G.close()


def test_reduced_errors():
    from paper_1712_02443_b200 import AimError
    G, R, O = setup("c1")
    eo, grp = G.elements()
    bad = type_blocks([10], ratio=2, seed=1)
    with pytest.raises(AimError) as e:
        G.reduced_set(grp, bad)              # block size != element size
    assert e.value.status == -1
    with pytest.raises(AimError):
        G.reduced_set(grp[:-1], type_blocks([288], ratio=2, seed=1))   # element count
    G.close()
