"""D15 GMRES parity at full size on configs C2-C5 (
PAPER.md:510-511; BASELINE.json north_star "GMRES solutions to <= 1e-5
relative error at equal iteration counts ... on all five configs").

The reference iterates were written by tools/make_goldens.py, which calls
only oracle/ (oracle GMRES: MGS + one reorthogonalisation, on the oracle's
own AIM operator with its radix-2 FFT) on the plane-wave right-hand side of
D14.  The oracle cannot reach the converged counts of C2/C3 (4164 / 2183
GMRES(50) iterations on the GPU) in CPU-hours, so the protocol runs both
sides for the same fixed count k -- two restart cycles on C2/C3, one cycle
(D15's k = 50) on C4/C5 -- and compares:
  * J_k on a stratified row sample (every grid x-plane, uniform rows) and
    through a 32-entry Gaussian sketch (relative L2 estimate), <= 1e-5;
  * the per-iteration residual estimate |g_{j+1}|/||V||, <= 1e-6 relative;
  * the true relative residual of J_k, <= 1e-6 relative;
  * the right-hand side V on the sampled rows (<= 1e-13);
  * the residual V - Z J_k of the GPU's J_k on sampled rows, recomputed with
    the oracle's row-sampled matvec (matvec_rows, pinned in
    tests/test_oracle_aim.py), against the GPU product's, <= 1e-8 ||V||.
"""
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from workloads import get_config, make_mesh  # noqa: E402
from workloads.sketch import sketch  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    path = os.path.join(GOLD, f"gmres_{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not written yet (tools/make_goldens.py)")
    d = np.load(path)
    return json.loads(str(d["meta"])), d


@pytest.mark.parametrize("name", ["c2", "c3", "c5", "c4"])
def test_gmres_golden_full_size(name):
    from paper_1712_02443_b200 import AimPlan
    meta, g = _golden(name)
    cfg = get_config(name)
    mesh = make_mesh(cfg)
    G = AimPlan.from_mesh(mesh, cfg.k, cfg.h, cfg.M, cfg.near_radius)
    assert G.N == meta["N"]
    V = G.planewave_rhs()
    rows = g["rows"]
    Vh = V.cpu().numpy()
    assert np.abs(Vh[rows] - g["V_rows"]).max() <= 1e-13 * np.abs(g["V_rows"]).max()
    k = meta["iters"]
    J, it, rr, _ = G.gmres(V, restart=meta["restart"], tol=meta["tol"], fixed_iters=k)
    assert it == k
    Jh = J.cpu().numpy()
    Jr = g["J_rows"]
    assert np.linalg.norm(Jh[rows] - Jr) <= 1e-5 * np.linalg.norm(Jr)
    s_ref = g["J_sketch"]
    s_gpu = sketch(Jh)
    assert np.linalg.norm(s_gpu - s_ref) <= 1e-5 * np.linalg.norm(s_ref)
    assert abs(np.linalg.norm(Jh) - float(g["jnorm"])) <= 1e-5 * float(g["jnorm"])
    assert abs(rr - meta["rel_res"]) <= 1e-6 * meta["rel_res"]
    # GPU residual of its own J vs the oracle's row-sampled product of that J
    ZJ = G.matvec(J).cpu().numpy()
    G.close()
    del J, V
    torch.cuda.empty_cache()
    from oracle.aim import OraclePlan
    O = OraclePlan(mesh, cfg.k, cfg.h, cfg.M, cfg.near_radius)
    sub = rows[np.linspace(0, rows.size - 1, 192).astype(np.int64)]
    r_gpu = Vh[sub] - ZJ[sub]
    r_ora = Vh[sub] - O.matvec_rows(Jh, sub, method="fft")
    assert np.linalg.norm(r_gpu - r_ora) <= 1e-8 * np.linalg.norm(Vh[sub])


def _arnoldi_lstsq(matvec, V, k):
    """Plain PyTorch GMRES reference of the same operation (one cycle of k
    steps, no restart): Arnoldi with modified Gram-Schmidt applied twice, then
    the (j+1) x j Hessenberg least-squares problems solved densely on the host
    (numpy lstsq) -- no Givens recurrences, nothing shared with k_gmres.cu.
    Returns J_k and |beta e1 - H_j y_j| / beta for j = 1..k."""
    beta = torch.linalg.vector_norm(V)
    Q = torch.empty((k + 1, V.numel()), dtype=V.dtype, device=V.device)
    H = np.zeros((k + 1, k), dtype=np.complex128)
    Q[0] = V / beta
    for j in range(k):
        w = matvec(Q[j]).clone()
        for _ in range(2):
            for i in range(j + 1):
                h = torch.vdot(Q[i], w)
                w -= h * Q[i]
                H[i, j] += complex(h)
        hn = torch.linalg.vector_norm(w)
        H[j + 1, j] = float(hn)
        Q[j + 1] = w / hn
    b = float(beta)
    hist = []
    y = None
    for j in range(1, k + 1):
        e1 = np.zeros(j + 1, dtype=np.complex128)
        e1[0] = b
        y, *_ = np.linalg.lstsq(H[:j + 1, :j], e1, rcond=None)
        hist.append(np.linalg.norm(e1 - H[:j + 1, :j] @ y) / b)
    J = (torch.as_tensor(y, device=V.device)[:, None] * Q[:k]).sum(0)
    return J, np.asarray(hist)


def test_gmres_c4_one_cycle():
    """C4 (BASELINE.json configs[3], the GMRES(50) workload) at D15's k = 50.
    The oracle's full C4 solve is out of reach (its near matrix alone is about
    13 core-hours, each product about 80 s), so no golden file exists for C4
    and the golden test above skips it.  Here the device solver is held to
      * a plain PyTorch Arnoldi + dense least-squares GMRES of the same k on
        the same operator: J_k <= 1e-5, the residual history <= 1e-6 relative;
      * GMRES's defining property at any size: r_k = V - Z J_k is orthogonal to
        Z K_k (checked against Z V and Z J_k, both in Z K_k);
      * the oracle: V on the stratified rows (<= 1e-13), and, with
        AIM_TEST_SLOW=1 (about 6 CPU-minutes), the residual of the GPU's J_k on
        sampled rows recomputed with the oracle's row-sampled product
        (matvec_rows, pinned in tests/test_oracle_aim.py), <= 1e-8 ||V||.
    The operator itself is compared with the oracle on >= 1,000 stratified
    rows in tests/test_gpu_parity.py."""
    from paper_1712_02443_b200 import AimPlan
    from workloads.sketch import stratified_rows
    cfg = get_config("c4")
    mesh = make_mesh(cfg)
    G = AimPlan.from_mesh(mesh, cfg.k, cfg.h, cfg.M, cfg.near_radius)
    V = G.planewave_rhs()
    k = 50
    J, it, rr, _ = G.gmres(V, restart=50, tol=1e-4, fixed_iters=k)
    assert it == k
    hist = G.gmres_history()
    assert hist.size == k
    Jref, href = _arnoldi_lstsq(G.matvec, V, k)
    assert float(torch.linalg.vector_norm(J - Jref)) <= 1e-5 * float(torch.linalg.vector_norm(Jref))
    assert np.abs(hist - href).max() <= 1e-6 * href.min()
    del Jref
    ZJ = G.matvec(J)
    r = V - ZJ
    bn = float(torch.linalg.vector_norm(V))
    rn = float(torch.linalg.vector_norm(r))
    assert abs(rn / bn - rr) <= 1e-6 * rr
    assert abs(rn / bn - hist[-1]) <= 1e-6 * rr
    ZV = G.matvec(V)
    for Zv in (ZV, ZJ):
        assert abs(complex(torch.vdot(Zv, r))) <= 1e-8 * float(torch.linalg.vector_norm(Zv)) * rn
    Vh, Jh, ZJh = V.cpu().numpy(), J.cpu().numpy(), ZJ.cpu().numpy()
    G.close()
    del J, V, ZJ, ZV, r
    torch.cuda.empty_cache()
    from oracle.efie import EfieContext
    from oracle.excitation import plane_wave_rhs
    from oracle.aim import stencil_bases
    ctx = EfieContext(mesh.vertices, mesh.triangles, mesh.rwg, cfg.k)
    rows = stratified_rows(stencil_bases(ctx.geo["centre"], cfg.h, cfg.M), n_random=1024, seed=7)
    Vo = plane_wave_rhs(ctx)
    assert np.abs(Vh[rows] - Vo[rows]).max() <= 1e-13 * np.abs(Vo).max()
    if os.environ.get("AIM_TEST_SLOW") != "1":
        return      # the oracle's C4 plan + one FFT product of J_k take about 6 CPU-minutes
    from oracle.aim import OraclePlan
    O = OraclePlan(mesh, cfg.k, cfg.h, cfg.M, cfg.near_radius)
    sub = rows[np.linspace(0, rows.size - 1, 192).astype(np.int64)]
    r_gpu = Vh[sub] - ZJh[sub]
    r_ora = Vo[sub] - O.matvec_rows(Jh, sub, method="fft")
    assert np.linalg.norm(r_gpu - r_ora) <= 1e-8 * np.linalg.norm(Vh[sub])
