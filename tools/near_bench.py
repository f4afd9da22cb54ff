"""Time the H6 near-field kernels alone on one config (CUDA events, per kernel
choice via AIM_NEAR_KERNEL).   python tools/near_bench.py [config] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1712_02443_b200 import AimPlan  # noqa: E402
from workloads import get_config, make_mesh, make_vectors  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg = get_config(name)
plan = AimPlan.from_mesh(make_mesh(cfg), cfg.k, cfg.h, cfg.M, cfg.near_radius)
x = torch.from_numpy(make_vectors(plan.N, cfg.nrhs, 0)).cuda()
ys = {}
for kern in ("mma", "b4", "csr"):
    os.environ["AIM_NEAR_KERNEL"] = kern
    for _ in range(3):
        y = plan.interpolate(None, x, add_near=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        y = plan.interpolate(None, x, add_near=True)
    e1.record()
    torch.cuda.synchronize()
    ys[kern] = y
    print(f"{name} near {kern}: {e0.elapsed_time(e1) / reps * 1e3:.1f} us  lib={os.environ.get('AIM_LIB', 'default')}")
d = (ys["mma"] - ys["csr"]).norm() / ys["csr"].norm()
print(f"mma vs csr rel {float(d):.2e}")
