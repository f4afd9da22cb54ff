"""A/B of the near SpMV beside the FFT (k_near_stream.cu) against the in-order
near1 product: unprofiled CUDA-event time per product, bitwise comparison.
    python tools/ovl_ab.py c4 [steps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import timed_steps  # noqa: E402
from paper_1712_02443_b200 import AimPlan  # noqa: E402
from workloads import get_config, make_mesh, make_vectors  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
cfg = get_config(name)
mesh = make_mesh(cfg)
x = torch.from_numpy(make_vectors(mesh.n_rwg, 1, 0)[:, 0].copy()).cuda()
out = {"config": name}
ref = None
ALL = {"off": {}, "prio128": {"AIM_NEAR_PRIO": "1"}, "prio256": {"AIM_NEAR_PRIO": "1", "AIM_NEAR_PRIO_T": "256"},
       "prio256_nc": {"AIM_NEAR_PRIO": "1", "AIM_NEAR_PRIO_T": "256", "AIM_NEAR_CARVE": "0", "AIM_NEAR1_CARVE": "0"},
       "prio256_fc": {"AIM_NEAR_PRIO": "1", "AIM_NEAR_PRIO_T": "256", "AIM_NEAR1_CARVE": "0"},
       "prio128_nc": {"AIM_NEAR_PRIO": "1", "AIM_NEAR_CARVE": "0", "AIM_NEAR1_CARVE": "0"},
       "prio128_fc": {"AIM_NEAR_PRIO": "1", "AIM_NEAR1_CARVE": "0"},
       "ovl_a1f10": {"AIM_NEAR_OVL": "1", "AIM_NEAR_OVL_A": "1", "AIM_NEAR_OVL_F": "0.1"}}
names = sys.argv[3].split(",") if len(sys.argv) > 3 else ["off", "prio128", "prio256", "ovl_a1f10", "off"]
variants = [(n, ALL[n]) for n in names]
plan = AimPlan.from_mesh(mesh, cfg.k, cfg.h, cfg.M, cfg.near_radius)
for tag, env in variants:
    for k in ("AIM_NEAR_OVL", "AIM_NEAR_OVL_A", "AIM_NEAR_OVL_F", "AIM_NEAR_PRIO", "AIM_NEAR_PRIO_T", "AIM_NEAR_CARVE",
              "AIM_NEAR1_CARVE"):
        os.environ.pop(k, None)
    os.environ.update(env)
    plan.compress(0)                   # drops the captured graphs
    y = plan.matvec(x)
    if ref is None:
        ref = y.clone()
    t, _ = timed_steps(lambda: plan.matvec(x, y), steps, 3)
    out[tag + ("" if tag not in out else "_2")] = {"ms": 1e3 * t / steps, "bitwise_equal_to_off": bool(torch.equal(y, ref))}
    print(tag, out[tag], flush=True)
print(json.dumps(out), flush=True)
plan.close()
