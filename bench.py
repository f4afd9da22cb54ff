#!/usr/bin/env python
"""Benchmark of the AIM matvec hot path (BASELINE.json metric: AIM matvecs/sec,
complex128, and fraction of the HBM roofline).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]
                  [--replicas] [--no-extra] [--no-cpu-baseline]

Workload (default): BASELINE.json configs[3] = "c4", the 32x32 array of
0.5-lambda cubes (N = 1,843,200 RWG unknowns), h = 0.05, M = 3, near radius
0.2; one step = one single-RHS aim_matvec (the product GMRES(50) applies on
this config): near-field SpMV, projection, the FFT convolution passes and the
interpolation.  `value` = matvecs per second.

N = 1: one plan on one GPU.  N > 1 (torchrun, one process per GPU): the
slab-decomposed operator (aim_slab_*; x-slabs, NCCL all-to-all FFT
transposes, strong scaling: the ranks cooperate on every product), or with
--replicas one independent plan per GPU (weak scaling, no collective).

Timing: CUDA events on the launching stream around exactly K steps after
W >= 3 warm-up steps, barrier + synchronize on both sides, max over ranks.
The headline loop runs with profiling off; per-stage times come from a
separate profiled pass (events recorded by the library between its kernels
on the kernel's stream).  Inputs exceed the 126 MB L2 (C4: near matrix 9.6 GB,
weights 7.5 GB), so no L2 flush is needed.

Extra objects on the line (rank 0, N = 1): `roofline` (dominant kernel,
algorithmic bytes per launch / its event-timed duration vs the measured HBM
copy peak), `matvec_roofline` (SURVEY.md §8(d) compulsory bytes per product),
`e2e` (aim_matvec_host_steps: host x in, host y out every step, copies
overlapped inside the library), `cufft` (cuFFT Z2Z on the same zero-padded
4-component 3-D convolution, a comparison baseline only), `configs` (C2 16 RHS,
C3, C5 complex128, C5 complex64, each with its own clock record),
`cpu_baseline` (the CPU oracle on a bounded sample, 1 core and all cores).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "AIM matvecs/sec (complex128)"
UNIT = "matvecs/s"
BASELINE_INDEX = {"c1": 0, "c2": 1, "c3": 2, "c4": 3, "c5": 4}


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def workload_label(cfg, N, R, prec="c128"):
    dims = "x".join(str(d) for d in cfg.shape)
    idx = BASELINE_INDEX.get(cfg.name)
    src = f"BASELINE.json configs[{idx}]" if idx is not None else "test case"
    return f"{cfg.name}: {src} ({dims} array, N={N}, {R} RHS, {prec})"


def alg_bytes(info, R, es=16):
    """Compulsory (algorithmic) bytes per matvec and per
    launch of each stage kernel, for R right-hand sides and element size es
    (16 complex128, 8 complex64; weights 8 or 4 bytes)."""
    ws = es // 2
    N, S, Ng = info["n_rwg"], info["S"], info["n_nodes"]
    nnzP, nnzN = info["nnz_proj"], info["nnz_near"]
    Px, Py, Pz = info["fft_dims"]
    Nx, Ny, Nz = info["grid_dims"]
    spec = es * (Px // 2 + 1) * (Py // 2 + 1) * (Nz if info["conv_mode"] != 0 else Pz // 2 + 1)
    grid = 4 * es * Ng * R                               # one 4-component grid, R RHS
    xpad = 4 * es * Px * Ny * Nz * R                     # x-padded grid
    matvec = (es * N * R + (4 * ws + 4) * nnzP + 4 * (Ng + 1) + 4 * grid + spec
              + 4 * ws * nnzP + 4 * N + (es + 4) * nnzN + 8 * (N + 1) + es * N * R)
    stages = {
        "near": (es + 4) * nnzN + 8 * (N + 1) + es * N * R + es * N * R,       # Z, col, rowptr, x, y
        "project": (4 * ws + 4) * nnzP + 4 * (Ng + 1) + es * N * R + grid,     # w + n, rowptr, x, Q
        "interp": 4 * ws * nnzP + 4 * N + grid + 2 * es * N * R,               # w, base, Phi, y (r+w)
        "fft_x": grid + xpad,                                                  # Q -> W1
        "fft_yz": 2 * xpad + spec,                                             # W1 -> W1 + spectrum
        "ifft_x": xpad + grid,                                                 # W1 -> Phi
    }
    return matvec, stages


def alg_bytes_compressed(info, ci, R=1, es=16):
    """Compulsory bytes of the repetition-compressed product (NEXT-3): the
    vectors, the four grid passes and the spectrum as alg_bytes, the near
    dictionary (value + column) and the projection templates (4 weights + row)
    read once, and per RWG its grid node and weight-row index (single RHS)."""
    N, Ng = info["n_rwg"], info["n_nodes"]
    Px, Py, Pz = info["fft_dims"]
    Nz = info["grid_dims"][2]
    spec = es * (Px // 2 + 1) * (Py // 2 + 1) * (Nz if info["conv_mode"] != 0 else Pz // 2 + 1)
    grid = 4 * es * Ng * R
    return (2 * es * N * R + 4 * grid + spec + (es + 4) * ci["dict_nnz"] + (4 * es // 2 + 4) * ci.get("tpl_nnz", 0)
            + 8 * N)


def fp64_peak():
    """FP64 FMA peak derived from the unit counts and clock (148 SMs x 64 FP64
    lanes x 2 flop x 1.965 GHz; tools/fp64_peak.cu measures 34.2 TFLOP/s)."""
    return 148 * 64 * 2 * 1.965e9 / 1e12, "derived: 148 SM x 64 FP64 lanes x 2 x 1.965 GHz"


def planar_flops(info, R):
    Px, Py, _ = info["fft_dims"]
    Nz = info["grid_dims"][2]
    lines = 4 * Px * Nz * R
    return 2 * lines * 5 * Py * math.log2(Py) + 4 * Px * Py * R * 8 * Nz * Nz


def kernel_names(info, R):
    mode = info["conv_mode"]
    return {
        "near": ("near1_kernel (H6 near-field SpMV, warp per row)" if R == 1 else
                 "near_mma_kernel (H6 near-field SpMM, FP64 tensor cores)" if R >= 8 else "near_b4/near_kernel (H6)"),
        "project": "project1_kernel (H1 projection gather)" if R == 1 else "project_kernel (H1 projection gather)",
        "interp": "interp1_kernel (H5 interpolation)" if R == 1 else "interp_kernel (H5 interpolation)",
        "fft_x": "fft_ct/fft_pp kernel (H2 x forward, zero-pad fused)",
        "fft_yz": {1: "planar4_kernel (y fwd, z Toeplitz x G2, y inv, fused)",
                   2: "ymode2_kernel (y fwd, z Toeplitz x G2, y inv fused; TMA bulk copies)" if R == 1
                   else "y passes + ztoeplitz_kernel (mode 2)",
                   0: "fft passes y fwd, z turnaround x G, y inv"}[mode],
        "ifft_x": "fft_ct/fft_pp kernel (H4 x inverse, pruned)",
    }


def load_traffic(cfg_name, stage):
    """DRAM bytes per launch of the stage's kernel from the committed ncu
    --set full capture (profiles/traffic_<config>.json), if any."""
    path = os.path.join(ROOT, "profiles", f"traffic_{cfg_name}.json")
    if os.path.exists(path):
        return json.load(open(path)).get(stage)
    return None


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(device_index), f"--query-gpu=timestamp,{self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "20"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
        self.f.flush()
        rows = [l.split(",") for l in open(self.f.name).read().strip().splitlines() if l.count(",") >= 7]
        os.unlink(self.f.name)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if "Active" in r[4 + i] and "Not" not in r[4 + i]})
        busy = [v for v in sm if v > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    return ws, rank, local


def max_over_ranks(t, ws):
    if ws == 1:
        return t
    import torch
    tt = torch.tensor([t], dtype=torch.float64, device="cuda")
    torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
    return float(tt.item())


# ---------------------------------------------------------------- GPU timing
def timed_steps(fn, steps, warmup, ws=1, clocks_dev=None, preheat_s=0.3):
    """W warm-up calls (plus a short pre-heat so the clock sampler sees load),
    then exactly `steps` calls between CUDA events on the current stream,
    barrier + synchronize on both sides; returns (seconds max over ranks, clocks)."""
    import torch
    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    clk = ClockSampler(clocks_dev) if clocks_dev is not None else None
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < preheat_s:
        fn()
        torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(steps):
        fn()
    ev1.record(stream)
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    clocks = clk.stop() if clk else None
    return max_over_ranks(ev0.elapsed_time(ev1) / 1e3, ws), clocks


def profile_stages(plan, x, y, reps):
    """Per-stage milliseconds from a separate profiled pass (library events)."""
    import torch
    plan.profile(True)
    for _ in range(reps):
        plan.matvec(x, y)
    torch.cuda.synchronize()
    st, n = plan.profile_read()
    plan.profile(False)
    return {k: v / max(1, n) for k, v in st.items()}


def cufft_compare(info, R, ours_conv_ms, reps=10):
    """cuFFT (torch.fft, complex128 Z2Z) on the same zero-padded 4-component
    convolution: forward 3-D FFT with padding, x spectrum, inverse, pruned
    copy back -- timed only as a comparison baseline (north_star)."""
    import torch
    Nx, Ny, Nz = info["grid_dims"]
    Px, Py, Pz = info["fft_dims"]
    if info["conv_mode"] != 0:
        Pz = 2 * Nz - 1                 # planar modes do z directly; cuFFT pads it
    shape = (4, Nx, Ny, Nz) + ((R,) if R > 1 else ())
    g = torch.Generator(device="cuda").manual_seed(0)
    Q = torch.randn(shape, dtype=torch.complex128, device="cuda", generator=g)
    G = torch.randn((Px, Py, Pz) + ((1,) if R > 1 else ()), dtype=torch.complex128, device="cuda", generator=g)
    Phi = torch.empty_like(Q)

    def step():
        F = torch.fft.fftn(Q, s=(Px, Py, Pz), dim=(1, 2, 3))
        F *= G
        Phi.copy_(torch.fft.ifftn(F, dim=(1, 2, 3))[:, :Nx, :Ny, :Nz])

    t, _ = timed_steps(step, reps, 2, preheat_s=0.0)
    ms = 1e3 * t / reps
    out = {"ms_per_convolution": ms, "ours_ms_per_convolution": ours_conv_ms,
           "speedup_ours_vs_cufft": ms / ours_conv_ms if ours_conv_ms else None,
           "padded": [Px, Py, Pz], "what": "torch.fft.fftn/ifftn (cuFFT Z2Z) on [4][Nx][Ny][Nz][R] zero-padded to "
                                           "[Px][Py][Pz], times a spectrum, pruned copy; ours = fft_x + fft_yz + ifft_x"}
    del Q, G, Phi
    torch.cuda.empty_cache()
    return out


def measure_extras(plan, x, y, steps, warmup, local, gm_iters=50):
    """On the headline plan (one RHS): GMRES per-iteration cost (D15; CGS2
    vector passes beside the product), the block-Jacobi preconditioner
    (NEXT-4: build time, preconditioned iteration cost), the reduced
    macromodel system product (NEXT-2, seeded synthetic blocks of the paper's
    shapes, N_m = 4 N^_m) and the repetition-compressed near field (NEXT-3)."""
    import numpy as np
    import torch
    from workloads.macromodel import type_blocks
    out = {}
    V = plan.planewave_rhs()
    plan.gmres(V, restart=50, tol=1e-12, fixed_iters=2)      # workspace (Krylov basis) allocated untimed
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, it, rr, _ = plan.gmres(V, restart=50, tol=1e-12, fixed_iters=gm_iters)
    t_gm = time.perf_counter() - t0
    mv_ms = None
    t, _ = timed_steps(lambda: plan.matvec(x, y), 10, 2, preheat_s=0.0)
    mv_ms = 1e3 * t / 10
    gm = {"iters": it, "ms_per_iter": 1e3 * t_gm / it, "matvec_ms": mv_ms,
          "vector_ms_per_iter": 1e3 * t_gm / it - mv_ms * (1 + 1.0 / 50),
          "what": f"GMRES(50), {gm_iters} fixed iterations from J0 = 0 on the D14 plane wave (one true-residual "
                  "product per restart cycle included), host wall clock around aim_gmres"}
    t0 = time.perf_counter()
    pc = plan.precond_build(1)
    pc["build_seconds"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    _, it, _, _ = plan.gmres(V, restart=50, tol=1e-12, fixed_iters=gm_iters)
    pc["ms_per_iter"] = 1e3 * (time.perf_counter() - t0) / it
    plan.precond_build(0)
    gm["block_jacobi"] = pc
    out["gmres"] = gm
    eo, grp = plan.elements()
    sizes = [int((eo == e).sum()) for e in [list(grp).index(d) for d in range(int(grp.max()) + 1)]]
    if len(sizes) <= 4:
        blocks = type_blocks(sizes, ratio=4, seed=11)
        t0 = time.perf_counter()
        plan.reduced_set(grp, blocks)
        t_set = time.perf_counter() - t0
        del blocks
        ry = torch.empty_like(x)
        t, _ = timed_steps(lambda: plan.reduced_matvec(x, ry), 10, 2, preheat_s=0.0)
        out["reduced"] = {"ms_per_product": 1e3 * t / 10, "products_per_s": 10 / t, "set_seconds": t_set,
                          "types": len(sizes), "elements": int(grp.size), "nhat": sizes, "nint": [4 * s for s in sizes],
                          "what": "(D - G T A^-1 B) Y, PAPER.md eq. MV_product1: two per-type block GEMMs (D, "
                                  "K = T A^-1 B, FP64) around one aim_matvec; seeded synthetic blocks"}
    t0 = time.perf_counter()
    ci = plan.compress(1)
    ci["build_seconds"] = time.perf_counter() - t0
    t, clk = timed_steps(lambda: plan.matvec(x, y), steps, warmup, clocks_dev=local)
    b = alg_bytes_compressed(plan.info, ci)
    peak, peak_src = load_peaks()
    ci.update({"value": steps / t, "ms_per_step": 1e3 * t / steps, "clocks": clk,
               "stage_ms": profile_stages(plan, x, y, max(3, min(steps, 20))),
               "matvec_roofline": {"bound": "hbm", "alg_bytes": b, "achieved": b / (t / steps) / 1e9, "peak": peak,
                                   "unit": "GB/s", "frac": b / (t / steps) / 1e9 / peak, "peak_source": peak_src},
               "what": "repetition-compressed operators: near field from the dictionary (sparse x dense over "
                       "element pairs), projection through the group templates, interpolation with the "
                       "representative's weight rows; the FFT convolution as the headline"})
    plan.compress(0)
    out["compressed"] = ci
    return out


def measure_config(name, precision, steps, warmup, local, e2e_steps=0, cufft=False, extras=False):
    """One plan, one timed loop (profiling off), a profiled pass; returns a dict."""
    import numpy as np
    import torch
    from paper_1712_02443_b200 import AimPlan, launch_count
    from workloads import get_config, make_mesh, make_vectors
    cfg = get_config(name)
    mesh = make_mesh(cfg)
    R = cfg.nrhs
    plan = AimPlan.from_mesh(mesh, cfg.k, cfg.h, cfg.M, cfg.near_radius, precision=precision)
    info = plan.info
    xh = make_vectors(mesh.n_rwg, R, seed=0)
    if R == 1:
        xh = xh[:, 0].copy()
    xh = xh.astype(plan.np_dtype)
    x = torch.from_numpy(xh).cuda()
    y = torch.empty_like(x)
    t, clocks = timed_steps(lambda: plan.matvec(x, y), steps, warmup, clocks_dev=local)
    launch_count(reset=True)
    plan.matvec(x, y)
    launches = launch_count()           # kernels of one product (data-independent)
    stage_ms = profile_stages(plan, x, y, max(3, min(steps, 20)))
    es = 8 if precision == 1 else 16
    b_mv, b_stage = alg_bytes(info, R, es)
    peak, peak_src = load_peaks()
    ms = 1e3 * t / steps
    res = {"config": name, "workload": workload_label(cfg, info["n_rwg"], R, "c64" if precision else "c128"),
           "value": steps * R / t, "unit": UNIT, "ms_per_step": ms, "steps": steps, "nrhs": R,
           "matvec_roofline": {"bound": "hbm", "alg_bytes": b_mv, "achieved": b_mv / (ms / 1e3) / 1e9,
                               "peak": peak, "unit": "GB/s", "frac": b_mv / (ms / 1e3) / 1e9 / peak},
           "stage_ms": stage_ms,
           "stage_alg_gbs": {k: (b_stage[k] / (stage_ms[k] / 1e3) / 1e9 if stage_ms.get(k) else None)
                             for k in b_stage},
           "clocks": clocks, "plan_seconds": info["plan_seconds"], "device_bytes": info["device_bytes"],
           "grid": list(info["grid_dims"]), "fft": list(info["fft_dims"]), "conv_mode": info["conv_mode"],
           "nnz_proj": info["nnz_proj"], "nnz_near": info["nnz_near"]}
    res["_info"], res["_b_stage"], res["_launches_per_step"] = info, b_stage, launches
    if e2e_steps:
        # end to end through the C ABI with host buffers: every step copies its x
        # from pinned host memory and its y back; copies overlap neighbouring products
        xp = torch.from_numpy(xh).pin_memory().numpy()
        ys = [torch.from_numpy(np.empty_like(xh)).pin_memory().numpy() for _ in range(3)]
        plan.matvec_host_steps([xp] * 3, ys)
        t0 = time.perf_counter()
        plan.matvec_host_steps([xp] * e2e_steps, [ys[i % 3] for i in range(e2e_steps)])
        te = time.perf_counter() - t0
        ysync = np.empty_like(xh)
        plan.matvec_host(xp, ysync)
        t1 = time.perf_counter()
        for _ in range(max(3, e2e_steps // 4)):
            plan.matvec_host(xp, ysync)
        ts = (time.perf_counter() - t1) / max(3, e2e_steps // 4)
        res["e2e"] = {"value": e2e_steps * R / te, "unit": UNIT, "h2d_bytes_per_step": int(xh.nbytes),
                      "d2h_bytes_per_step": int(xh.nbytes), "steps": e2e_steps,
                      "timer": "host wall clock around aim_matvec_host_steps (C ABI): every step copies its x "
                               "from pinned host memory and its y back; step i's copy-in, step i-1's product "
                               "and step i-2's copy-out overlap on three streams",
                      "synchronous": {"value": R / ts, "timer": "host wall clock, aim_matvec_host per step "
                                                                 "(copy in, product, copy out, synchronise)"}}
    if cufft:
        conv = sum(stage_ms.get(k, 0.0) for k in ("fft_x", "fft_yz", "ifft_x"))
        res["cufft"] = cufft_compare(info, R, conv)
    if extras and R == 1 and precision == 0:
        res.update(measure_extras(plan, x, y, steps, warmup, local))
    plan.close()
    torch.cuda.empty_cache()
    return res


def roofline_of(res, name):
    info, b_stage, stage_ms = res["_info"], res["_b_stage"], res["stage_ms"]
    R = res["nrhs"]
    peak, peak_src = load_peaks()
    dom = max(b_stage, key=lambda k: stage_ms.get(k, 0.0))
    ms = stage_ms[dom]
    timing = ("CUDA events recorded by the library around the kernel on its launch stream, averaged over a "
              "profiled pass of the same products (the headline loop runs unprofiled)")
    names = kernel_names(info, R)
    share = ms / res["ms_per_step"]
    if dom == "fft_yz" and info["conv_mode"] == 1:
        fl = planar_flops(info, R)
        pk, pk_src = fp64_peak()
        tf = fl / (ms / 1e3) / 1e12
        return {"kernel": names[dom], "stage": dom, "bound": "alu", "achieved": tf, "peak": pk,
                "unit": "TFLOP/s", "frac": tf / pk, "traffic": load_traffic(name, dom),
                "alg_flops_per_launch": fl, "alg_bytes_per_launch": b_stage[dom], "ms_per_launch": ms,
                "share_of_step": share, "peak_source": pk_src, "timing": timing}
    ach = b_stage[dom] / (ms / 1e3) / 1e9
    return {"kernel": names[dom], "stage": dom, "bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
            "frac": ach / peak, "traffic": load_traffic(name, dom), "alg_bytes_per_launch": b_stage[dom],
            "ms_per_launch": ms, "share_of_step": share, "peak_source": peak_src, "timing": timing}


# ----------------------------------------------------------- CPU oracle sample
_OS = {}


def _os_near(rows):
    import numpy as np
    Z = _OS["O"].near_matrix(np.asarray(rows))
    return Z


def _os_work(item):
    """One part of the bounded oracle sample (runs in-process or in a worker)."""
    import numpy as np
    from oracle.fft import fft_radix2
    kind, a, b = item
    O, x = _OS["O"], _OS["x"]
    if kind == "near":
        _OS["Z"][a:b] @ x[_OS["cols"]]   # rows [a, b) of the sampled near rows
    elif kind == "proj":
        for P in _OS["P"]:
            P[:, a:b] @ x[_OS["prow"][a:b]]
    elif kind == "interp":
        O.interpolate(_OS["Phi"], _OS["irow"][a:b])
    elif kind == "fft":
        ax, n = a, b
        fft_radix2(_OS["lines"][ax][:n], axis=-1)
        fft_radix2(_OS["lines"][ax][:n], axis=-1, inverse=True)
    elif kind == "mul":
        _OS["mul"][a:b] * _OS["mul"][a:b]
    return 0


def oracle_sample(cfg, mesh, workers_list=(1, None), near_rows=1024, frac=None):
    """The oracle (oracle/aim.py, as it stands) timed on a BOUNDED sample of
    the workload, on 1 host core and on all host cores (fork pool):

      near     Z_corr rows @ x for `near_rows` evenly spaced rows (rows built
               untimed), scaled by N / near_rows;
      far      a fraction f of the far-field work, scaled by 1/f: projection
               over f N columns of P, interpolation of f N rows, f of the
               radix-2 FFT lines of the 9 padded 3-D transforms of one product
               (4 components x forward + inverse + the kernel spectrum
               convolve_fft recomputes) and f of the spectrum products.
    Returns the cpu_baseline object (value for all cores; the 1-core run
    inside)."""
    import numpy as np
    import scipy.sparse as sp
    from multiprocessing import get_context
    from oracle.aim import OraclePlan
    from workloads import make_vectors
    ncores = os.cpu_count() or 1
    t0 = time.perf_counter()
    O = OraclePlan(mesh, cfg.k, cfg.h, cfg.M, cfg.near_radius)
    N = O.N
    x = make_vectors(N, 1, 0)
    pads = tuple(int(2 ** np.ceil(np.log2(2 * d - 1))) if d > 1 else 1 for d in O.dims)
    npad = int(np.prod(pads))
    if frac is None:
        frac = min(1.0, 3.0e6 / npad)          # ~10 s of single-core work at C4 size
    rows = np.linspace(0, N - 1, near_rows).astype(np.int64)
    _OS.clear()
    _OS.update(O=O, x=x)
    ctx = get_context("fork")
    with ctx.Pool(min(ncores, 16)) as pool:
        parts = pool.map(_os_near, np.array_split(rows, min(ncores, 16)))
    Z = sp.vstack(parts).tocsr()
    cols = np.unique(Z.indices)
    Zc = sp.csr_matrix((Z.data, np.searchsorted(cols, Z.indices), Z.indptr), shape=(Z.shape[0], cols.size))
    nf = max(1, int(round(frac * N)))
    prow = np.linspace(0, N - 1, nf).astype(np.int64)
    nodes = O.stencil_nodes(prow)
    colidx = np.repeat(np.arange(nf), O.S)
    P = [sp.csr_matrix((O.W[prow][:, :, c].ravel(), (nodes.ravel(), colidx)), shape=(O.Ng, nf)).tocsc()
         for c in range(4)]
    rng = np.random.default_rng(0)
    Phi = (rng.standard_normal((4,) + tuple(O.dims) + (1,)) + 0j)
    lines = []
    line_counts = []
    for a in range(3):
        total_lines = npad // pads[a] * 9
        n = max(1, int(round(frac * total_lines)))
        lines.append(np.ones((n, pads[a]), dtype=np.complex128))
        line_counts.append(n)
    nmul = max(1, int(round(frac * npad * 4)))
    _OS.update(Z=Zc, cols=cols, P=P, prow=prow, Phi=Phi, irow=prow, lines=lines,
               mul=np.ones(nmul, dtype=np.complex128))
    setup_s = time.perf_counter() - t0

    def items(k):
        out_near = [("near", int(s[0]), int(s[-1]) + 1) for s in np.array_split(np.arange(near_rows), k) if s.size]
        out_far = []
        for s in np.array_split(np.arange(nf), k):
            if s.size:
                out_far += [("proj", int(s[0]), int(s[-1]) + 1), ("interp", int(s[0]), int(s[-1]) + 1)]
        for a in range(3):
            for s in np.array_split(np.arange(line_counts[a]), k):
                if s.size:
                    out_far.append(("fft", a, int(s.size)))
        for s in np.array_split(np.arange(nmul), k):
            if s.size:
                out_far.append(("mul", int(s[0]), int(s[-1]) + 1))
        return out_near, out_far

    runs = {}
    for w in workers_list:
        k = ncores if w is None else w
        near_items, far_items = items(k)
        if k == 1:
            best = None
            for _ in range(1):
                a = time.perf_counter()
                for it in near_items:
                    _os_work(it)
                b = time.perf_counter()
                for it in far_items:
                    _os_work(it)
                c = time.perf_counter()
                cand = (b - a, c - b)
                best = cand if best is None else (min(best[0], cand[0]), min(best[1], cand[1]))
        else:
            with ctx.Pool(k) as pool:
                pool.map(_os_work, [("mul", 0, 1)] * k)          # workers up
                best = None
                for _ in range(2):
                    a = time.perf_counter()
                    pool.map(_os_work, near_items, chunksize=1)
                    b = time.perf_counter()
                    pool.map(_os_work, far_items, chunksize=1)
                    c = time.perf_counter()
                    cand = (b - a, c - b)
                    best = cand if best is None else (min(best[0], cand[0]), min(best[1], cand[1]))
        t_mv = best[0] * N / near_rows + best[1] / frac
        runs[k] = {"value": 1.0 / t_mv, "seconds_per_matvec": t_mv, "cores": k,
                   "sample_seconds": best[0] + best[1]}
    kmax = max(runs)
    res = {"value": runs[kmax]["value"], "unit": UNIT, "cores": kmax, "kind": "oracle", "host_cores": ncores,
           "seconds_per_matvec": runs[kmax]["seconds_per_matvec"],
           "one_core": runs.get(1),
           "sample": (f"{cfg.name} (N={N}, one RHS): near-field SpMV on {near_rows} evenly spaced rows scaled by "
                      f"N/{near_rows}; far field on a fraction f={frac:.4f} (projection over fN columns, "
                      f"interpolation of fN rows, f of the radix-2 FFT lines of the 9 power-of-two padded "
                      f"{pads} transforms, f of the spectrum products) scaled by 1/f; best of 2 (1 core: one "
                      f"run); numpy/scipy "
                      f"in {kmax} processes (fork pool) and in 1"),
           "setup_seconds": setup_s}
    _OS.clear()
    return res


def run_reference(args, ws, rank):
    """--impl reference: the CPU oracle (the paper has no code) on the box's
    host cores, on this arm's config and metric; rank 0 only."""
    if rank != 0:
        return
    from workloads import get_config, make_mesh
    cfg = get_config(args.config)
    mesh = make_mesh(cfg)
    cb = oracle_sample(cfg, mesh)
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": ws,
            "steps": 2, "warmup": 0, "ms_per_step": 1e3 * cb["seconds_per_matvec"],
            "higher_is_better": True, "scaling": "strong" if ws > 1 else "weak", "vs_baseline": None,
            "dtype": "c128", "data": "synthetic (seeded cube-array mesh, N(0,1) vectors)",
            "config": {"workload": workload_label(cfg, mesh.n_rwg, 1)},
            "cpu_baseline": cb, "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                                         "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- slab (N > 1)
def run_slab(args, ws, rank, local):
    """The slab-decomposed operator (aim_slab_*), one rank per GPU over NCCL
    (at N = 1 a one-rank communicator), strong scaling of one product."""
    import torch
    from paper_1712_02443_b200 import AimSlabPlan, launch_count, nccl_unique_id
    from paper_1712_02443_b200.api import slab_nccl_id
    from workloads import get_config, make_mesh, make_vectors

    torch.cuda.set_device(local)
    cfg = get_config(args.config)
    mesh = make_mesh(cfg)
    R = cfg.nrhs
    nid = slab_nccl_id() if ws > 1 else nccl_unique_id()
    t0 = time.perf_counter()
    plan = AimSlabPlan.from_mesh(mesh, cfg.k, cfg.h, cfg.M, cfg.near_radius, ws, rank, nid)
    plan_s = time.perf_counter() - t0
    q = plan.query(rank)
    xh = make_vectors(mesh.n_rwg, R, seed=0)
    if R == 1:
        xh = xh[:, 0].copy()
    x = torch.from_numpy(xh).cuda()
    y = torch.empty_like(x)
    t, clocks = timed_steps(lambda: plan.matvec(x, y), args.steps, args.warmup, ws,
                            clocks_dev=local if rank == 0 else None)
    launch_count(reset=True)
    plan.matvec(x, y)
    launches = launch_count() * args.steps
    value = args.steps * R / t
    xp = torch.from_numpy(xh).pin_memory()
    yp = torch.empty_like(xp).pin_memory()
    torch.distributed.barrier() if ws > 1 else None
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        x.copy_(xp, non_blocking=True)
        plan.matvec(x, y)
        yp.copy_(y, non_blocking=True)
        torch.cuda.synchronize()
    te = max_over_ranks(time.perf_counter() - t0, ws)
    peak, peak_src = load_peaks()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "c128", "data": "synthetic (seeded cube-array mesh per BASELINE.json, N(0,1) complex vectors)",
        "config": {"workload": workload_label(cfg, mesh.n_rwg, R) + f", slab-decomposed over {ws} GPU(s)",
                   "N": mesh.n_rwg, "nrhs": R, "parallelism": f"x-slabs x{ws} (NCCL all-to-all FFT transposes)",
                   "slab_rank0": q, "l2": "inputs > 126 MB L2 (no flush needed)"},
        "nvlink": {"a2a_bytes_per_rank_per_step": q["a2a_bytes_per_rhs"] * R,
                   "halo_bytes_per_rank_per_step": q["halo_bytes_per_rhs"] * R},
        "e2e": {"value": args.e2e_steps * R / te, "unit": UNIT, "h2d_bytes_per_step": int(xh.nbytes),
                "d2h_bytes_per_step": int(xh.nbytes), "steps": args.e2e_steps,
                "timer": "host wall clock around copy + product + copy, max over ranks"},
        "gpu_launches": int(launches),
        "clocks": clocks, "plan_seconds": plan_s, "peak_hbm_gbs": peak, "peak_source": peak_src,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    plan.close()
    if ws > 1:
        torch.distributed.destroy_process_group()


# ---------------------------------------------------------------- main path
def run_ours(args, ws, rank, local):
    import torch
    from paper_1712_02443_b200 import AimPlan, launch_count
    from workloads import get_config, make_mesh, make_vectors
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    torch.cuda.set_device(local)
    cfg = get_config(args.config)
    N1 = ws == 1
    head = measure_config(args.config, 0, args.steps, args.warmup, local, e2e_steps=args.e2e_steps if N1 else 0,
                          cufft=N1, extras=N1 and not args.no_extra) if N1 else None
    if not N1:
        # --replicas: one independent plan per GPU on its own input (weak scaling)
        mesh = make_mesh(cfg)
        plan = AimPlan.from_mesh(mesh, cfg.k, cfg.h, cfg.M, cfg.near_radius)
        R = cfg.nrhs
        xh = make_vectors(mesh.n_rwg, R, seed=rank)
        x = torch.from_numpy(xh[:, 0].copy() if R == 1 else xh).cuda()
        y = torch.empty_like(x)
        t, clocks = timed_steps(lambda: plan.matvec(x, y), args.steps, args.warmup, ws,
                                clocks_dev=local if rank == 0 else None)
        launch_count(reset=True)
        plan.matvec(x, y)
        head = {"value": ws * args.steps * R / t, "ms_per_step": 1e3 * t / args.steps, "clocks": clocks,
                "_launches_per_step": launch_count(), "workload": workload_label(cfg, mesh.n_rwg, R)}
        plan.close()
    per_step_launches = head["_launches_per_step"]
    line = {
        "metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic (seeded cube-array mesh per BASELINE.json, N(0,1) complex vectors)",
        "config": {"workload": head["workload"], "parallelism": f"rhs-replicas x{ws}" if ws > 1 else "1 GPU",
                   "l2": "inputs > 126 MB L2 (near matrix + weights); no flush needed"},
        "gpu_launches": int(round(per_step_launches * args.steps)),
        "clocks": head["clocks"],
    }
    if N1:
        line["config"].update({k: head[k] for k in ("grid", "fft", "conv_mode", "nnz_proj", "nnz_near", "nrhs")})
        line["config"]["N"] = head["_info"]["n_rwg"]
        line["roofline"] = roofline_of(head, args.config)
        for k in ("matvec_roofline", "stage_ms", "stage_alg_gbs", "e2e", "cufft", "plan_seconds", "device_bytes",
                  "gmres", "reduced", "compressed"):
            if k in head:
                line[k] = head[k]
        if not args.no_extra:
            extra = {}
            for name, prec in (("c2", 0), ("c3", 0), ("c5", 0), ("c5", 1)):
                if name == args.config and prec == 0:
                    continue
                r = measure_config(name, prec, max(10, min(args.steps, 50)), args.warmup, local)
                r["roofline"] = roofline_of(r, name)
                for k in [k for k in r if k.startswith("_")]:
                    r.pop(k)
                extra[f"{name}_{'c64' if prec else 'c128'}"] = r
            line["configs"] = extra
        if not args.no_cpu_baseline:
            line["cpu_baseline"] = oracle_sample(cfg, make_mesh(cfg))
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the per-config lines (C2, C3, C5 c128/c64)")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: independent plans per GPU (weak scaling) instead of the slab decomposition")
    ap.add_argument("--slab", action="store_true", help="slab-decomposed operator also at N = 1")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    ws, rank, local = dist_init()
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    if args.slab or (ws > 1 and not args.replicas):
        run_slab(args, ws, rank, local)
        return
    run_ours(args, ws, rank, local)


if __name__ == "__main__":
    main()
