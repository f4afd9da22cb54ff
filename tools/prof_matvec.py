"""Run a few matvecs of one config (for ncu / compute-sanitizer captures).
    python tools/prof_matvec.py [config] [nmatvec] [cmp]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1712_02443_b200 import AimPlan  # noqa: E402
from workloads import get_config, make_mesh, make_vectors  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
nmv = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = get_config(name)
mesh = make_mesh(cfg)
plan = AimPlan.from_mesh(mesh, cfg.k, cfg.h, cfg.M, cfg.near_radius)
x = torch.from_numpy(make_vectors(mesh.n_rwg, cfg.nrhs, 0)).cuda()
if "cmp" in sys.argv[3:]:          # the repetition-compressed operators, single RHS
    plan.compress(1)
    x = x[:, 0].contiguous()
for _ in range(nmv):
    y = plan.matvec(x)
torch.cuda.synchronize()
print(name, plan.info["n_rwg"], float(y.abs().sum()))
