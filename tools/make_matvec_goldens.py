"""Write the full-size matvec golden files tests/golden/matvec_<config>.npz from
the CPU oracle ONLY (eqs. AIM_step1-3 plus the precorrected
near rows).  Nothing here touches the CUDA path: the file
imports oracle/ and workloads/ and nothing else of the repo.

    python tools/make_matvec_goldens.py <config> [nrhs]

For config c (BASELINE.json configs, workloads.CONFIGS) it builds the oracle
plan, draws the seeded input x = workloads.make_vectors(N, nrhs, 0) (the vector
the GPU tests and bench.py use), picks the stratified row sample
(workloads.sketch.stratified_rows on the oracle's stencil bases: one RWG per
grid x-plane, 32 of each D3 tie class, two on either side of every cut of the
x-planes into 8 equal slabs, the first and last row, uniform rows; >= 1,000
rows, >= 500 for the 16-RHS C2) and stores OraclePlan.matvec_rows(x, rows) --
the full projection, the oracle's own radix-2 FFT convolution, interpolation
and exact near rows of the sampled rows.  tests/test_gpu_parity.py compares the
CUDA product with these values; with AIM_TEST_SLOW=1 it recomputes them live.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.aim import OraclePlan  # noqa: E402
from workloads import get_config, make_mesh, make_vectors  # noqa: E402
from workloads.sketch import stratified_rows  # noqa: E402


def golden_rows(O, cfg, n_random, min_rows):
    t = O.centres / cfg.h - (cfg.M - 1) / 2.0
    tie = np.abs(t - np.round(t)) <= 1e-6
    nx = int(O.bases[:, 0].max() - O.bases[:, 0].min()) + 1
    cuts = [int(round(nx * r / 8)) for r in range(1, 8)]
    while True:
        rows = stratified_rows(O.bases, n_random=n_random, seed=3, slab_bounds=cuts, tie_mask=tie)
        if rows.size >= min_rows:
            return rows
        n_random += min_rows - rows.size + 16


def main():
    name = sys.argv[1]
    nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    cfg = get_config(name)
    mesh = make_mesh(cfg)
    t0 = time.time()
    O = OraclePlan(mesh, cfg.k, cfg.h, cfg.M, cfg.near_radius)
    x = make_vectors(O.N, nrhs, 0)
    rows = golden_rows(O, cfg, 640 if nrhs == 1 else 400, 1000 if nrhs == 1 else 500)
    method = "fft" if nrhs == 1 else "auto"
    ref = O.matvec_rows(x, rows, method=method)
    meta = {"config": name, "N": int(O.N), "nrhs": nrhs, "x_seed": 0, "method": method, "rows": int(rows.size),
            "x_planes": int(np.unique(O.bases[:, 0]).size), "x_planes_covered": int(np.unique(O.bases[rows, 0]).size),
            "writer": "tools/make_matvec_goldens.py (oracle only)", "oracle_seconds": time.time() - t0,
            "reading": "PAPER.md:539-559; SURVEY.md §8(c)"}
    out = os.path.join(ROOT, "tests", "golden", f"matvec_{name}.npz")
    np.savez_compressed(out, meta=json.dumps(meta), rows=rows, ref=ref)
    print(json.dumps(meta), flush=True)


if __name__ == "__main__":
    main()
