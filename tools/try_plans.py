"""Create a plan + one matvec for each named config (quick GPU smoke of the launch paths)."""
import os
import sys
import traceback

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1712_02443_b200 import AimPlan  # noqa: E402
from workloads import get_config, make_mesh, make_vectors  # noqa: E402

for name in sys.argv[1:]:
    cfg = get_config(name)
    try:
        plan = AimPlan.from_mesh(make_mesh(cfg), cfg.k, cfg.h, cfg.M, cfg.near_radius)
        x = torch.from_numpy(make_vectors(plan.N, cfg.nrhs, 0)).cuda()
        y = plan.matvec(x)
        torch.cuda.synchronize()
        print(name, "ok", plan.info["fft_dims"], plan.info["conv_mode"], float(y.abs().sum()))
        plan.close()
    except Exception:
        print(name, "FAILED")
        traceback.print_exc()
