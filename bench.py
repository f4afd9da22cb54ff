#!/usr/bin/env python
"""Benchmark of the AIM matvec hot path (BASELINE.json metric: AIM matvecs/sec,
complex128, and fraction of the HBM roofline).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference] [--slab]

Workload (default): BASELINE.json configs[1] = "c2", the 10x10 array of
0.4-lambda cubes (N = 115,200 RWG unknowns), h = 0.05, M = 2, near radius 0.2,
batched matvec on 16 seeded complex128 N(0,1) vectors.  One step = one
aim_matvec on the 16-RHS batch (projection, 5 FFT passes, interpolation +
near-field SpMV).  `value` counts single-RHS matvecs per second over all
ranks.  N > 1: one process per GPU, each rank runs an independent replica
plan on its own 16-RHS batch (RHS sharding, no data-path collective, weak
scaling).  --slab: the slab-decomposed operator
(default config c4, the 1.8M-unknown array): the ranks cooperate on every
product (x-slabs, NCCL all-to-all FFT transposes, strong scaling).

Timing: CUDA events on the launching stream, W warm-up steps, barrier +
synchronize on both sides, max over ranks.  The working set (near matrix
600 MB, weights 100 MB, grids 0.85 GB) exceeds the 126 MB L2, so no L2 flush is
needed between steps.  Stage times come from CUDA events recorded by the
library between its kernels inside the timed region (aim_profile).
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


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def alg_bytes(info, R):
    """Compulsory (algorithmic) bytes per matvec and per
    launch of each stage kernel, for R right-hand sides."""
    N, S, Ng = info["n_rwg"], info["S"], info["n_nodes"]
    nnzP, nnzN = info["nnz_proj"], info["nnz_near"]
    Px, Py, Pz = info["fft_dims"]
    Nx, Ny, Nz = info["grid_dims"]
    spec = 16 * (Px // 2 + 1) * (Py // 2 + 1) * (Nz if info["conv_mode"] != 0 else Pz // 2 + 1)
    matvec = (16 * N * R + 36 * nnzP + 4 * (Ng + 1) + 4 * 64 * Ng * R + spec
              + 32 * nnzP + 4 * N + 20 * nnzN + 4 * (N + 1) + 16 * N * R)
    grid = 64 * Ng * R                                   # one 4-component grid, R RHS
    xpad = 64 * Px * Ny * Nz * R                         # x-padded grid
    stages = {
        "near": 20 * nnzN + 8 * (N + 1) + 16 * N * R + 16 * N * R,          # Z, col, rowptr, x, y
        "project": 36 * nnzP + 4 * (Ng + 1) + 16 * N * R + grid,            # ent+w, rowptr, x, Q
        "interp": 32 * nnzP + 4 * N + grid + 2 * 16 * N * R,                # w, base, Phi, y (r+w)
        "fft_x": grid + xpad,                                              # Q -> W1
        "fft_yz": 2 * xpad + spec,                                         # W1 in place + spectrum
        "ifft_x": xpad + grid,                                             # W1 -> Phi
    }
    return matvec, stages


def fp64_peak():
    """FP64 FMA peak derived from the unit counts and clock (B200: 148 SMs x 64
    FP64 lanes per clock x 2 flop x 1.965 GHz max SM clock).
    tools/fp64_peak.cu measured 34.2 TFLOP/s for a DFMA loop (profiles/fp64_peak.txt)."""
    return 148 * 64 * 2 * 1.965e9 / 1e12, "derived: 148 SM x 64 FP64 lanes x 2 x 1.965 GHz"


def planar_flops(info, R):
    """Algorithmic flops of one planar y/z launch: forward + inverse y FFTs of
    length Py over 4 Px Nz R lines (5 P log2 P each) and the direct z Toeplitz
    product, 8 Nz^2 flops per (component, kx, ky, rhs) column."""
    Px, Py, _ = info["fft_dims"]
    Nz = info["grid_dims"][2]
    lines = 4 * Px * Nz * R
    return 2 * lines * 5 * Py * math.log2(Py) + 4 * Px * Py * R * 8 * Nz * Nz


KERNEL_NAMES = {
    "near": "near_mma_kernel (H6 precorrected near-field SpMM, FP64 tensor cores)",
    "project": "project_kernel (H1 projection gather)",
    "interp": "interp_kernel (H5 interpolation)",
    "fft_x": "fft_ct_kernel (x forward, zero-pad fused)",
    "fft_yz": "planar4_kernel (y fwd FFT, z Toeplitz x G2, y inv FFT, fused)",
    "ifft_x": "fft_ct_kernel (x inverse, pruned)",
}


def load_traffic(stage):
    """DRAM bytes per launch of the stage's kernel from the committed ncu
    capture (profiles/traffic_c2.json: dram__bytes_read.sum + write), if any."""
    path = os.path.join(ROOT, "profiles", "traffic_c2.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return d.get(stage)
    return None


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(device_index), f"--query-gpu=timestamp,{self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "50"], stdout=self.f,
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


def oracle_sample(cfg, mesh, x, near_rows=1024, reps=2):
    """The oracle as it stands on a bounded sample of the workload: the full
    far field (projection, power-of-two FFT convolution, interpolation) for one
    RHS, and the precorrected near-field product for `near_rows` evenly spaced
    rows (its near matrix built untimed, like the GPU plan), extrapolated to
    all N rows.  numpy/scipy run these single-threaded."""
    import numpy as np
    from oracle.aim import OraclePlan
    O = OraclePlan(mesh, cfg.k, cfg.h, cfg.M, cfg.near_radius)
    rows = np.linspace(0, O.N - 1, near_rows).astype(np.int64)
    Nr = O.near_matrix(rows)
    x1 = x[:, :1]
    O.far(x1, "fft")   # warm (projection matrices)
    tf, tn = [], []
    for _ in range(reps):
        t0 = time.perf_counter()
        O.far(x1, "fft")
        t1 = time.perf_counter()
        Nr @ x1
        t2 = time.perf_counter()
        tf.append(t1 - t0)
        tn.append(t2 - t1)
    t_mv = min(tf) + min(tn) * O.N / rows.size
    return {"value": 1.0 / t_mv, "unit": UNIT, "cores": 1, "kind": "oracle",
            "host_cores": os.cpu_count(),
            "sample": (f"{cfg.name}: 1 of {cfg.nrhs} RHS; far field over the full grid "
                       f"(oracle power-of-two FFT); near SpMV on {rows.size} of {O.N} rows extrapolated to N; "
                       f"best of {reps}; numpy/scipy single-threaded"),
            "seconds_per_matvec": t_mv}


def run_reference(args, ws, rank):
    """--impl reference: the oracle (the paper has no code) timed on host cores."""
    if rank != 0:
        return
    import numpy as np
    from workloads import get_config, make_mesh, make_vectors
    cfg = get_config(args.config)
    mesh = make_mesh(cfg)
    x = make_vectors(mesh.n_rwg, cfg.nrhs, 0)
    steps = max(1, min(args.steps, 5))
    cb = oracle_sample(cfg, mesh, x, reps=steps)
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": ws,
            "steps": steps, "warmup": 1, "ms_per_step": 1e3 * cb["seconds_per_matvec"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128",
            "data": "synthetic (seeded cube-array mesh, N(0,1) vectors)",
            "config": {"workload": f"{cfg.name}: BASELINE.json configs[1] (10x10 array, N=115200, 16 RHS)"},
            "cpu_baseline": cb, "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                                         "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_slab(args, ws, rank, local):
    """--slab: the slab-decomposed operator (aim_slab_*), one rank per GPU over
    NCCL (at N = 1 a one-rank communicator), strong scaling of one product."""
    import numpy as np
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
    xh = make_vectors(mesh.n_rwg, R, seed=0)          # x replicated on every rank
    x = torch.from_numpy(xh).cuda()
    y = torch.empty_like(x)
    stream = torch.cuda.current_stream()

    def barrier():
        if ws > 1:
            torch.distributed.barrier()

    for _ in range(args.warmup):
        plan.matvec(x, y)
    torch.cuda.synchronize()
    barrier()
    clk = ClockSampler(local) if rank == 0 else None
    time.sleep(0.15 if clk else 0)
    torch.cuda.synchronize()
    barrier()
    launch_count(reset=True)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        plan.matvec(x, y)
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    launches = launch_count()
    clocks = clk.stop() if clk else None
    t = ev0.elapsed_time(ev1) / 1e3
    if ws > 1:
        tt = torch.tensor([t], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t = float(tt.item())
    value = args.steps * R / t                        # one product per step for the whole job
    # end to end: pinned host x -> device, product, y -> pinned host, every step
    xp = torch.from_numpy(xh).pin_memory()
    yp = torch.empty_like(xp).pin_memory()
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        x.copy_(xp, non_blocking=True)
        plan.matvec(x, y)
        yp.copy_(y, non_blocking=True)
        torch.cuda.synchronize()
    te = time.perf_counter() - t0
    if ws > 1:
        tt = torch.tensor([te], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        te = float(tt.item())
    ms_step = 1e3 * t / args.steps
    peak, peak_src = load_peaks()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "c128", "data": "synthetic (seeded cube-array mesh per BASELINE.json, N(0,1) complex vectors)",
        "config": {"workload": f"{cfg.name}: slab-decomposed product (N={mesh.n_rwg}, {R} RHS)",
                   "N": mesh.n_rwg, "nrhs": R, "parallelism": f"x-slabs x{ws} (NCCL all-to-all FFT transposes)",
                   "slab_rank0": q, "l2": "working set > 126 MB L2 (no flush needed)"},
        "nvlink": {"a2a_bytes_per_rank_per_step": q["a2a_bytes_per_rhs"] * R,
                   "halo_bytes_per_rank_per_step": q["halo_bytes_per_rhs"] * R},
        "e2e": {"value": args.e2e_steps * R / te, "unit": UNIT, "h2d_bytes_per_step": int(xh.nbytes),
                "d2h_bytes_per_step": int(xh.nbytes), "steps": args.e2e_steps,
                "timer": "host wall clock around copy + product + copy"},
        "gpu_launches": int(launches), "clocks": clocks, "plan_seconds": plan_s, "peak_hbm_gbs": peak,
        "peak_source": peak_src,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    plan.close()
    if ws > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--slab", action="store_true",
                    help="slab-decomposed operator over the ranks (default config c4) instead of RHS replicas")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.slab and "--config" not in sys.argv:
        args.config = "c4"
    ws, rank, local = dist_init()
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    if args.slab:
        run_slab(args, ws, rank, local)
        return

    import numpy as np
    import torch
    from paper_1712_02443_b200 import AimPlan, launch_count
    from workloads import get_config, make_mesh, make_vectors

    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    torch.cuda.set_device(local)
    cfg = get_config(args.config)
    mesh = make_mesh(cfg)
    R = cfg.nrhs
    plan = AimPlan.from_mesh(mesh, cfg.k, cfg.h, cfg.M, cfg.near_radius)
    info = plan.info
    xh = make_vectors(mesh.n_rwg, R, seed=rank)
    x = torch.from_numpy(xh).cuda()
    y = torch.empty_like(x)
    stream = torch.cuda.current_stream()

    def barrier():
        if ws > 1:
            torch.distributed.barrier()

    for _ in range(args.warmup):
        plan.matvec(x, y)
    torch.cuda.synchronize()
    barrier()
    clk = ClockSampler(local) if rank == 0 else None
    time.sleep(0.15 if clk else 0)
    torch.cuda.synchronize()
    barrier()
    launch_count(reset=True)
    plan.profile(True)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        plan.matvec(x, y)
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    launches = launch_count()
    stages, nprof = plan.profile_read()
    plan.profile(False)
    clocks = clk.stop() if clk else None
    t = ev0.elapsed_time(ev1) / 1e3
    if ws > 1:
        tt = torch.tensor([t], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t = float(tt.item())
    value = ws * args.steps * R / t

    # end-to-end through the C ABI with host buffers (pinned), copies timed
    xp = torch.from_numpy(xh).pin_memory().numpy()
    yp = torch.empty_like(torch.from_numpy(xh)).pin_memory().numpy()
    for _ in range(2):
        plan.matvec_host(xp, yp)
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        plan.matvec_host(xp, yp)
    te = time.perf_counter() - t0
    if ws > 1:
        tt = torch.tensor([te], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        te = float(tt.item())
    e2e_sync = {"value": ws * args.e2e_steps * R / te, "steps": args.e2e_steps,
                "timer": "host wall clock, synchronous aim_matvec_host per step"}
    # pipelined: step i's x copy-in, step i-1's product and step i-2's y copy-out overlap
    from paper_1712_02443_b200.api import HostPipeline
    hp = HostPipeline(plan, R)
    xpt = torch.from_numpy(xh).pin_memory()
    ypt = [torch.empty_like(xpt).pin_memory() for _ in range(2)]
    for i in range(4):
        hp.submit(xpt, ypt[i % 2])
    hp.drain()
    barrier()
    n_e2e = max(args.e2e_steps, 50)
    t0 = time.perf_counter()
    for i in range(n_e2e):
        hp.submit(xpt, ypt[i % 2])
    hp.drain()
    tp = time.perf_counter() - t0
    if ws > 1:
        tt = torch.tensor([tp], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        tp = float(tt.item())
    e2e = {"value": ws * n_e2e * R / tp, "unit": UNIT, "h2d_bytes_per_step": int(xh.nbytes),
           "d2h_bytes_per_step": int(xh.nbytes), "steps": n_e2e,
           "timer": "host wall clock over all steps; every step copies its x from pinned host memory and "
                    "its y back (HostPipeline: copies of neighbouring steps overlap the product)",
           "synchronous": e2e_sync}

    peak, peak_src = load_peaks()
    b_mv, b_stage = alg_bytes(info, R)
    stage_ms = {k: v / max(1, nprof) for k, v in stages.items()}
    stage_gbs = {k: (b_stage[k] / (stage_ms[k] / 1e3) / 1e9 if stage_ms.get(k) else None) for k in b_stage}
    dom = max(b_stage, key=lambda k: stage_ms.get(k, 0.0))
    ach = stage_gbs[dom]
    traffic = load_traffic(dom)
    timing = ("CUDA events recorded by the library around the kernel on its launch stream, "
              "averaged over the timed region")
    if dom == "fft_yz" and info["conv_mode"] == 1:
        # the fused planar y/z kernel is FP64-ALU bound (ncu: fp64 pipe busiest, DRAM ~10%)
        fl = planar_flops(info, R)
        pk, pk_src = fp64_peak()
        tf = fl / (stage_ms[dom] / 1e3) / 1e12
        roof = {"kernel": KERNEL_NAMES[dom], "bound": "alu", "achieved": tf, "peak": pk, "unit": "TFLOP/s",
                "frac": tf / pk, "traffic": traffic, "alg_flops_per_launch": fl,
                "alg_bytes_per_launch": b_stage[dom], "hbm_frac": ach / peak,
                "ms_per_launch": stage_ms[dom], "peak_source": pk_src, "timing": timing}
    else:
        roof = {"kernel": KERNEL_NAMES[dom], "bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                "frac": ach / peak, "traffic": traffic, "alg_bytes_per_launch": b_stage[dom],
                "ms_per_launch": stage_ms[dom], "peak_source": peak_src, "timing": timing}
    ms_step = 1e3 * t / args.steps
    mv_ach = b_mv / (ms_step / 1e3) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic (seeded cube-array mesh per BASELINE.json, N(0,1) complex vectors)",
        "config": {"workload": f"{cfg.name}: BASELINE.json configs[1] (10x10 array, N={info['n_rwg']}, {R} RHS)",
                   "N": info["n_rwg"], "nrhs": R, "grid": list(info["grid_dims"]), "fft": list(info["fft_dims"]),
                   "nnz_proj": info["nnz_proj"], "nnz_near": info["nnz_near"],
                   "parallelism": f"rhs-replicas x{ws}" if ws > 1 else "1 GPU",
                   "l2": "working set > 126 MB L2 (no flush needed)"},
        "roofline": roof,
        "matvec_roofline": {"bound": "hbm", "alg_bytes": b_mv, "achieved": mv_ach, "peak": peak, "unit": "GB/s",
                            "frac": mv_ach / peak},
        "stage_ms": stage_ms, "stage_alg_gbs": stage_gbs,
        "e2e": e2e, "gpu_launches": int(launches), "clocks": clocks,
        "plan_seconds": info["plan_seconds"], "device_bytes": info["device_bytes"],
    }
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = oracle_sample(cfg, mesh, xh)
    if rank == 0:
        print(json.dumps(line), flush=True)
    plan.close()
    if ws > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
