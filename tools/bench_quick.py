"""Unprofiled product time of one config (CUDA events, 30 products) -- A/B of
scheduling knobs.    python tools/bench_quick.py c4"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1712_02443_b200 import AimPlan  # noqa: E402
from workloads import get_config, make_mesh, make_vectors  # noqa: E402

for name in sys.argv[1:]:
    cfg = get_config(name)
    plan = AimPlan.from_mesh(make_mesh(cfg), cfg.k, cfg.h, cfg.M, cfg.near_radius)
    x = torch.from_numpy(make_vectors(plan.N, 1, 0)[:, 0].copy()).cuda()
    y = plan.matvec(x)
    y0 = y.clone()
    for _ in range(5):
        plan.matvec(x, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(30):
        plan.matvec(x, y)
    e1.record()
    torch.cuda.synchronize()
    print(name, os.environ.get("AIM_NEAR_SIDE", "-"), os.environ.get("AIM_NEAR_CTAS_PER_SM", "-"),
          "ms %.3f" % (e0.elapsed_time(e1) / 30), "equal", bool(torch.equal(y, y0)), flush=True)
    plan.close()
