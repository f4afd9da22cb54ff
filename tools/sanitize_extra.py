"""Small runs of the non-matvec device paths for compute-sanitizer: GMRES,
block-Jacobi build/apply, reduced system, compression, the mode-2 fused
kernel on a forced small grid is not compiled (C3/C4 sizes only)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1712_02443_b200 import AimPlan, AimSlabPlan  # noqa: E402
from workloads import get_config, make_mesh, make_vectors  # noqa: E402
from workloads.macromodel import type_blocks  # noqa: E402

cfg = get_config("t_vol")
mesh = make_mesh(cfg)
G = AimPlan.from_mesh(mesh, cfg.k, cfg.h, cfg.M, cfg.near_radius)
V = G.planewave_rhs()
G.gmres(V, restart=20, tol=1e-6, fixed_iters=25)
G.precond_build(1)
G.gmres(V, restart=20, tol=1e-6)
G.precond_build(0)
eo, grp = G.elements()
G.reduced_set(grp, type_blocks([int((eo == 0).sum())], ratio=2, seed=1))
G.reduced_matvec(V)
G.compress(1)
x = torch.from_numpy(make_vectors(G.N, 1, 0)[:, 0].copy()).cuda()
G.matvec(x)
G.matvec(x)
G.close()
S = AimSlabPlan.from_mesh(mesh, cfg.k, cfg.h, cfg.M, cfg.near_radius, 2)
S.matvec(x)
S.gmres(V, restart=20, tol=1e-6, fixed_iters=10)
S.close()
torch.cuda.synchronize()
print("sanitize_extra done")
