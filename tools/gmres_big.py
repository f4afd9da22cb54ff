"""GMRES(restart) on a large config (default C4: BASELINE.json configs[3],
plane wave D14, tol 1e-4): iterations, wall time, time per iteration.
    python tools/gmres_big.py [config] [restart] [tol] [max_iters]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1712_02443_b200 import AimPlan  # noqa: E402
from workloads import get_config, make_mesh  # noqa: E402

pre = "--precond" in sys.argv
sys.argv = [a for a in sys.argv if a != "--precond"]
name = sys.argv[1] if len(sys.argv) > 1 else "c4"
restart = int(sys.argv[2]) if len(sys.argv) > 2 else 50
tol = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-4
max_iters = int(sys.argv[4]) if len(sys.argv) > 4 else 20000
cfg = get_config(name)
plan = AimPlan.from_mesh(make_mesh(cfg), cfg.k, cfg.h, cfg.M, cfg.near_radius)
pc = {}
if pre:
    t0 = time.perf_counter()
    pc = plan.precond_build(1)
    pc["build_seconds"] = time.perf_counter() - t0
V = plan.planewave_rhs()
x = V.clone()
y = plan.matvec(x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    plan.matvec(x, y)
e1.record()
torch.cuda.synchronize()
t_mv = e0.elapsed_time(e1) / 5 / 1e3
t0 = time.perf_counter()
J, it, rr, st = plan.gmres(V, restart=restart, tol=tol, max_iters=max_iters)
torch.cuda.synchronize()
t = time.perf_counter() - t0
print(json.dumps({"config": name, "N": plan.N, "restart": restart, "tol": tol, "status": st, "iters": it,
                  "rel_res": rr, "seconds": t, "ms_per_iter": 1e3 * t / max(it, 1), "matvec_ms": 1e3 * t_mv,
                  "plan_seconds": plan.info["plan_seconds"], "precond": pc}))
