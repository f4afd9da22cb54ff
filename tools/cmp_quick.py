"""A/B of the general and the repetition-compressed product on one config
(unprofiled CUDA-event time + per-stage profile), and GMRES per-iteration
cost beside the product.     python tools/cmp_quick.py c4 [gmres_iters]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import profile_stages, timed_steps  # noqa: E402
from paper_1712_02443_b200 import AimPlan  # noqa: E402
from workloads import get_config, make_mesh, make_vectors  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
gm_iters = int(sys.argv[2]) if len(sys.argv) > 2 else 0
cfg = get_config(name)
plan = AimPlan.from_mesh(make_mesh(cfg), cfg.k, cfg.h, cfg.M, cfg.near_radius)
x = torch.from_numpy(make_vectors(plan.N, 1, 0)[:, 0].copy()).cuda()
y = plan.matvec(x)
out = {"config": name}
t, _ = timed_steps(lambda: plan.matvec(x, y), 30, 3)
out["general_ms"] = 1e3 * t / 30
out["general_stages"] = profile_stages(plan, x, y, 5)
y0 = y.clone()
t0 = time.perf_counter()
out["compress"] = plan.compress(1)
out["compress_s"] = time.perf_counter() - t0
y1 = plan.matvec(x)
out["rel_vs_general"] = float((y1 - y0).norm() / y0.norm())
t, _ = timed_steps(lambda: plan.matvec(x, y), 30, 3)
out["compressed_ms"] = 1e3 * t / 30
out["compressed_stages"] = profile_stages(plan, x, y, 5)
os.environ["AIM_CMP_SIDE"] = "0"        # near in order (the graphs are rebuilt by compress)
plan.compress(1)
t, _ = timed_steps(lambda: plan.matvec(x, y), 30, 3)
out["compressed_in_order_ms"] = 1e3 * t / 30
del os.environ["AIM_CMP_SIDE"]
plan.compress(1)
if gm_iters:
    for mode in (0, 1):
        plan.compress(mode)
        V = plan.planewave_rhs()
        plan.gmres(V, restart=50, tol=1e-12, fixed_iters=2)
        t, _ = timed_steps(lambda: plan.matvec(x, y), 10, 2, preheat_s=0.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, it, rr, _ = plan.gmres(V, restart=50, tol=1e-12, fixed_iters=gm_iters)
        tg = time.perf_counter() - t0
        out[f"gmres_cmp{mode}"] = {"iters": it, "ms_per_iter": 1e3 * tg / it, "matvec_ms": 1e3 * t / 10,
                                   "vector_ms": 1e3 * tg / it - 1e3 * t / 10 * (1 + 1 / 50)}
print(json.dumps(out), flush=True)
plan.close()
