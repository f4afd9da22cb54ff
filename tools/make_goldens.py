"""Write the GMRES golden files tests/golden/gmres_<config>.npz from the CPU
oracle ONLY (reading D15).  Nothing here touches the CUDA
path: the file imports oracle/ and workloads/ and nothing else of the repo.

    python tools/make_goldens.py <config> <iterations> [workers]

For config c (BASELINE.json configs, workloads.CONFIGS) it builds the oracle
plan, then the oracle's full near matrix (OraclePlan.near_matrix over row
chunks in a process pool -- the same function on disjoint rows), and runs
oracle.gmres.gmres(restart=50, tol=1e-4, fixed_iters=<iterations>) on the
plane-wave right-hand side of D14 (oracle.excitation.plane_wave_rhs).  The
matvec is OraclePlan.matvec's steps (project -> convolve_fft -> interpolate,
plus the near matrix); the four grid components' FFT convolutions run in
parallel processes (convolve_fft treats them independently).

The golden file stores what the GPU test compares (tests/test_gpu_gmres.py):
iterations, the per-iteration residual estimate |g_{j+1}|/||V||, the true
relative residual of the returned iterate, ||V||, ||J||, J on a stratified
row sample (workloads.sketch.stratified_rows) and a 32-entry Gaussian sketch
of J (workloads.sketch.sketch), so the relative L2 error of the GPU's J can
be estimated without storing 10^6 entries.
"""
from __future__ import annotations

import json
import os
import sys
import time
from multiprocessing import get_context

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.aim import OraclePlan  # noqa: E402
from oracle.excitation import plane_wave_rhs  # noqa: E402
from oracle.gmres import gmres  # noqa: E402
from workloads import get_config, make_mesh  # noqa: E402
from workloads.sketch import sketch, stratified_rows  # noqa: E402

_O = None   # the oracle plan, inherited by the forked workers


def _near_chunk(rows):
    Z = _O.near_matrix(rows)
    return Z.data, Z.indices.astype(np.int32), np.diff(Z.indptr).astype(np.int32)


def _conv_component(Qc):
    return _O.convolve_fft(Qc)


def build_near(pool, N, nchunks):
    import scipy.sparse as sp
    bounds = np.linspace(0, N, nchunks + 1).astype(np.int64)
    parts = pool.map(_near_chunk, [np.arange(bounds[i], bounds[i + 1]) for i in range(nchunks)], chunksize=1)
    cnt = np.concatenate([p[2] for p in parts])
    indptr = np.zeros(N + 1, dtype=np.int64)
    np.cumsum(cnt, out=indptr[1:])
    data = np.concatenate([p[0] for p in parts])
    idx = np.concatenate([p[1] for p in parts])
    del parts
    return sp.csr_matrix((data, idx, indptr), shape=(N, N))


def main():
    global _O
    name = sys.argv[1]
    iters = int(sys.argv[2])
    workers = int(sys.argv[3]) if len(sys.argv) > 3 else max(1, (os.cpu_count() or 2) - 1)
    cfg = get_config(name)
    mesh = make_mesh(cfg)
    t0 = time.time()
    _O = OraclePlan(mesh, cfg.k, cfg.h, cfg.M, cfg.near_radius)
    ctx = get_context("fork")
    with ctx.Pool(workers) as pool:
        near = build_near(pool, _O.N, max(64, 8 * workers))
    _O._near = near
    t_plan = time.time() - t0
    print(f"{name}: N={_O.N} nnzN={near.nnz} oracle plan {t_plan:.0f}s", flush=True)

    V = plane_wave_rhs(_O.ctx)
    nmv = [0]
    with ctx.Pool(4) as pool:
        def matvec(x):
            x2 = np.asarray(x, dtype=np.complex128)[:, None]
            Q = _O.project(x2)
            Phi = np.concatenate(pool.map(_conv_component, [Q[c:c + 1] for c in range(4)]))
            nmv[0] += 1
            if nmv[0] % 5 == 0:
                print(f"  matvec {nmv[0]} at {time.time() - t0:.0f}s", flush=True)
            return (_O.interpolate(Phi) + near @ x2)[:, 0]

        t1 = time.time()
        res = gmres(matvec, V, restart=50, tol=1e-4, fixed_iters=iters)
        t_solve = time.time() - t1
    J = res["x"]
    rows = stratified_rows(_O.bases, n_random=1024, seed=7)
    out = os.path.join(ROOT, "tests", "golden", f"gmres_{name}.npz")
    meta = {"config": name, "N": int(_O.N), "restart": 50, "tol": 1e-4, "iters": int(res["iters"]),
            "rel_res": float(res["rel_res"]), "converged": bool(res["converged"]),
            "writer": "tools/make_goldens.py (oracle only)", "oracle_plan_s": t_plan, "oracle_solve_s": t_solve,
            "workers": workers, "reading": "D15 (SURVEY.md §8(c)); PAPER.md:510-511"}
    np.savez_compressed(out, meta=json.dumps(meta), history=np.asarray(res["history"]),
                        bnorm=np.linalg.norm(V), jnorm=np.linalg.norm(J), rows=rows, J_rows=J[rows],
                        J_sketch=sketch(J), V_rows=V[rows])
    print(json.dumps(meta), flush=True)


if __name__ == "__main__":
    main()
