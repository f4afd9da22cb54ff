"""Reduced-system product (PAPER.md eq. MV_product1) on a large config with
seeded synthetic macromodel blocks (workloads/macromodel.py): set-up time
and product time.    python tools/reduced_big.py [config] [ratio]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1712_02443_b200 import AimPlan  # noqa: E402
from workloads import get_config, make_mesh, make_vectors  # noqa: E402
from workloads.macromodel import type_blocks  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
ratio = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = get_config(name)
plan = AimPlan.from_mesh(make_mesh(cfg), cfg.k, cfg.h, cfg.M, cfg.near_radius)
eo, grp = plan.elements()
sizes = [int((eo == e).sum()) for e in [list(grp).index(d) for d in range(grp.max() + 1)]]
blocks = type_blocks(sizes, ratio=ratio, seed=11)
t0 = time.perf_counter()
plan.reduced_set(grp, blocks)
t_set = time.perf_counter() - t0
Y = torch.from_numpy(make_vectors(plan.N, 1, 0)[:, 0].copy()).cuda()
out = plan.reduced_matvec(Y)
x = plan.matvec(Y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
res = {}
for label, fn in (("reduced", lambda: plan.reduced_matvec(Y, out)), ("aim", lambda: plan.matvec(Y, x))):
    for _ in range(3):
        fn()
    e0.record()
    for _ in range(20):
        fn()
    e1.record()
    torch.cuda.synchronize()
    res[label + "_ms"] = e0.elapsed_time(e1) / 20
print(json.dumps({"config": name, "N": plan.N, "types": len(sizes), "elements": int(grp.size), "nhat": sizes[:4],
                  "ratio": ratio, "set_seconds": t_set, **res}))
