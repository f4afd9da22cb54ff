"""Diagnostic: slab product vs the single plan for nrhs sequences, fused and separate pack."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from workloads import get_config, make_mesh, make_vectors
from paper_1712_02443_b200 import AimPlan, AimSlabPlan, launch_count
name, world = sys.argv[1], int(sys.argv[2])
seq = [int(v) for v in sys.argv[3].split(",")]
order = sys.argv[4].split(",") if len(sys.argv) > 4 else ["1", "0"]
cfg = get_config(name); mesh = make_mesh(cfg)
single = AimPlan.from_mesh(mesh, cfg.k, cfg.h, cfg.M, cfg.near_radius)
xs = {r: torch.from_numpy(make_vectors(mesh.n_rwg, r, 11 + r)).cuda() for r in set(seq)}
y1 = {r: single.matvec(x) for r, x in xs.items()}
single.close()
slab = AimSlabPlan.from_mesh(mesh, cfg.k, cfg.h, cfg.M, cfg.near_radius, world)
for fuse in order:
    os.environ["AIM_SLAB_FUSE_PACK"] = fuse
    for r in seq:
        c0 = launch_count(); y = slab.matvec(xs[r]); n = launch_count() - c0
        print(f"fuse={fuse} R={r} launches={n} rel={float((y - y1[r]).norm() / y1[r].norm()):.3e}", flush=True)
