"""Create a slab plan (device-copy exchanges) for one config and compare one
matvec with the single-GPU plan.   python tools/slab_try.py [config] [world]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1712_02443_b200 import AimPlan, AimSlabPlan  # noqa: E402
from workloads import get_config, make_mesh, make_vectors  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
world = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = get_config(name)
mesh = make_mesh(cfg)
t = time.time()
slab = AimSlabPlan.from_mesh(mesh, cfg.k, cfg.h, cfg.M, cfg.near_radius, world)
print("slab plan", time.time() - t, [slab.query(r) for r in range(world)])
x = torch.from_numpy(make_vectors(mesh.n_rwg, cfg.nrhs, 0)).cuda()
yg = slab.matvec(x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    slab.matvec(x, yg)
e1.record()
torch.cuda.synchronize()
print("slab product ms (all slabs on this GPU, sequential):", e0.elapsed_time(e1) / 5)
single = AimPlan.from_mesh(mesh, cfg.k, cfg.h, cfg.M, cfg.near_radius)
y1 = single.matvec(x)
print("rel", float((yg - y1).norm() / y1.norm()))
