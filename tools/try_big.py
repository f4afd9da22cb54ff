"""Plan + matvec timing for the large configs (C3, C4, C5): plan seconds, memory, matvec ms."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1712_02443_b200 import AimPlan  # noqa: E402
from workloads import get_config, make_mesh, make_vectors  # noqa: E402

args = sys.argv[1:]
prec = 1 if "--c64" in args else 0          # AIM_C64 plans (reading D16)
cmp = "--compress" in args                     # repetition-compressed near field (NEXT-3)
for name in [a for a in args if not a.startswith("--")]:
    cfg = get_config(name)
    t0 = time.time()
    mesh = make_mesh(cfg)
    t1 = time.time()
    plan = AimPlan.from_mesh(mesh, cfg.k, cfg.h, cfg.M, cfg.near_radius, precision=prec)
    inf = plan.info
    if cmp:
        t2 = time.time()
        ci = plan.compress(1)
        print(name, "compress", ci, "%.2fs" % (time.time() - t2), flush=True)
    x = torch.from_numpy(make_vectors(plan.N, 1, 0)).to(plan.dtype).cuda()
    y = plan.matvec(x)
    torch.cuda.synchronize()
    plan.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        plan.matvec(x, y)
    e1.record()
    torch.cuda.synchronize()
    st, n = plan.profile_read()
    print(name + ("/c64" if prec else ""), "N", plan.N, "mesh %.1fs" % (t1 - t0), "plan %.2fs" % inf["plan_seconds"], "GB %.2f" % (inf["device_bytes"] / 1e9),
          "grid", inf["grid_dims"], "fft", inf["fft_dims"], "mode", inf["conv_mode"], "nnzN", inf["nnz_near"],
          "matvec ms %.3f" % (e0.elapsed_time(e1) / 10), {k: round(v / max(n, 1), 3) for k, v in st.items()}, flush=True)
    plan.close()
