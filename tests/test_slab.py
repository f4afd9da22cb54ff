"""Slab-decomposed product: the host partition on CPU
(including a world_size-2 gloo run of the multi-process plumbing), and on the
GPU the G-slab operator with device-copy exchanges vs the single-GPU plan
(<= 1e-13) and the oracle (<= 1e-10)."""
import os
import socket

import numpy as np
import pytest

from workloads import get_config, make_mesh, make_vectors


def _oracle_bases(mesh, h, M):
    from oracle.aim import grid_box, stencil_bases
    from oracle.geometry import rwg_geometry
    geo = rwg_geometry(mesh.vertices, mesh.triangles, mesh.rwg)
    b = stencil_bases(geo["centre"], h, M)
    return b, grid_box(b, M)


@pytest.mark.parametrize("name", ["c1", "t_m3", "t_dissim", "c2"])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_partition(name, world):
    from paper_1712_02443_b200 import AimError, slab_partition
    cfg = get_config(name)
    mesh = make_mesh(cfg)
    b, (origin, dims) = _oracle_bases(mesh, cfg.h, cfg.M)
    if world * cfg.M > dims[0]:
        with pytest.raises(AimError):
            slab_partition(mesh, cfg.h, cfg.M, world)
        return
    X, owner, nx = slab_partition(mesh, cfg.h, cfg.M, world)
    assert nx == dims[0]
    assert X[0] == 0 and X[-1] == nx
    assert np.all(np.diff(X) >= cfg.M)                      # halo reaches one neighbour only
    bx = b[:, 0] - origin[0]                                 # D3 bases (oracle)
    assert np.array_equal(owner, np.searchsorted(X, bx, side="right") - 1)
    cnt = np.bincount(owner, minlength=world)
    per_plane = np.bincount(bx, minlength=nx).max()
    assert cnt.max() <= mesh.n_rwg / world + per_plane      # balanced to one plane


def test_partition_rejects_too_many_slabs():
    from paper_1712_02443_b200 import AimError, slab_partition
    cfg = get_config("c1")
    with pytest.raises(AimError):
        slab_partition(make_mesh(cfg), cfg.h, cfg.M, 12)     # 12 * M > Nx = 12


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, name, q):
    import torch
    import torch.distributed as dist
    from paper_1712_02443_b200 import slab_partition
    from paper_1712_02443_b200.api import slab_nccl_id
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = get_config(name)
    mesh = make_mesh(cfg)
    nid = slab_nccl_id()                                     # rank 0 makes it, all receive it
    X, owner, nx = slab_partition(mesh, cfg.h, cfg.M, world)
    mine = torch.tensor([int((owner == rank).sum())], dtype=torch.int64)
    counts = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(counts, mine)
    xs = [torch.zeros(world + 1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(xs, torch.from_numpy(X.astype(np.int64)))
    ids = [None] * world
    dist.all_gather_object(ids, nid)
    # max-over-ranks timing reduction as bench.py does it
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    q.put((rank, [int(c) for c in counts], [x.tolist() for x in xs], len(set(ids)), len(nid), float(t)))
    dist.destroy_process_group()


def test_gloo_world2_partition_and_plumbing():
    import torch.multiprocessing as mp
    world, name = 2, "c2"
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_gloo_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    N = make_mesh(get_config(name)).n_rwg
    for rank, counts, xs, nids, idlen, tmax in res:
        assert sum(counts) == N                              # every RWG owned exactly once
        assert xs[0] == xs[1]                                # identical partition on every rank
        assert nids == 1 and idlen == 128                    # one NCCL id, broadcast
        assert tmax == float(world)
    assert res[0][1] == res[1][1]


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["planar", "planar2", "3d"])
@pytest.mark.parametrize("name,world,nrhs", [("c1", 2, 1), ("c1", 3, 5), ("c1", 6, 16), ("t_m3", 2, 2),
                                             ("t_dissim", 3, 9), ("t_vol", 2, 3)])
def test_slab_matvec_vs_single_and_oracle(name, world, nrhs, mode, monkeypatch):
    """planar: x pencils through the fused planar kernel (transposed 2-D
    spectrum); planar2 (AIM_CONV_MODE=2): x passes around the z Toeplitz
    kernel; 3d (AIM_CONV_MODE=0): y and z passes local, x turnaround on the
    pencils with the transposed octant."""
    import torch
    from conftest import oracle_plan
    from paper_1712_02443_b200 import AimPlan, AimSlabPlan
    cfg = get_config(name)
    mesh = make_mesh(cfg)
    if mode != "planar":
        monkeypatch.setenv("AIM_CONV_MODE", "0" if mode == "3d" else "2")
    single = AimPlan.from_mesh(mesh, cfg.k, cfg.h, cfg.M, cfg.near_radius)
    assert single.info["conv_mode"] == {"planar": 1, "planar2": 2, "3d": 0}[mode] or name == "t_vol"
    slab = AimSlabPlan.from_mesh(mesh, cfg.k, cfg.h, cfg.M, cfg.near_radius, world)
    q = [slab.query(r) for r in range(world)]
    assert q[0]["n0"] == 0 and q[-1]["n1"] == mesh.n_rwg
    assert sum(d["nnz_near"] for d in q) == single.info["nnz_near"]
    x = make_vectors(mesh.n_rwg, nrhs, 3)
    xt = torch.from_numpy(x).cuda()
    y1 = single.matvec(xt).cpu().numpy()
    yg = slab.matvec(xt).cpu().numpy()
    assert np.linalg.norm(yg - y1) / np.linalg.norm(y1) <= 1e-13
    ref = oracle_plan(name).matvec(x)
    assert np.linalg.norm(yg - ref) / np.linalg.norm(ref) <= 1e-10
    assert np.array_equal(slab.matvec(xt).cpu().numpy(), yg)     # deterministic
    slab.close()
    single.close()


@pytest.mark.gpu
@pytest.mark.parametrize("name,world", [("c1", 2), ("c1", 3), ("t_dissim", 3), ("t_vol", 2), ("c2", 4)])
def test_slab_rank_local_near_rows(name, world, monkeypatch):
    """Rank-local plan build: a one-rank-per-process rank builds near rows only
    for the RWGs it owns (aim_plan::near_keep).  AIM_SLAB_RANK_NEAR=1 makes the
    in-process slabs take each rank's rows from a base plan built that way;
    the product equals the single plan's to 1e-13 and the near rows add up to
    the full near matrix."""
    import torch
    from paper_1712_02443_b200 import AimPlan, AimSlabPlan
    cfg = get_config(name)
    mesh = make_mesh(cfg)
    single = AimPlan.from_mesh(mesh, cfg.k, cfg.h, cfg.M, cfg.near_radius)
    monkeypatch.setenv("AIM_SLAB_RANK_NEAR", "1")
    slab = AimSlabPlan.from_mesh(mesh, cfg.k, cfg.h, cfg.M, cfg.near_radius, world)
    q = [slab.query(r) for r in range(world)]
    assert sum(d["nnz_near"] for d in q) == single.info["nnz_near"]
    xt = torch.from_numpy(make_vectors(mesh.n_rwg, 2, 5)).cuda()
    y1 = single.matvec(xt)
    yg = slab.matvec(xt)
    assert float((yg - y1).norm() / y1.norm()) <= 1e-13
    slab.close()
    single.close()


@pytest.mark.gpu
def test_slab_matvec_c2_full_size():
    """C2 at full size over 4 and 8 slabs (device-copy exchanges): equal to the
    single-GPU plan to 1e-13 on all 16 RHS."""
    import torch
    from paper_1712_02443_b200 import AimPlan, AimSlabPlan
    cfg = get_config("c2")
    mesh = make_mesh(cfg)
    single = AimPlan.from_mesh(mesh, cfg.k, cfg.h, cfg.M, cfg.near_radius)
    x = torch.from_numpy(make_vectors(mesh.n_rwg, cfg.nrhs, 0)).cuda()
    y1 = single.matvec(x)
    single.close()
    for world in (4, 8):
        slab = AimSlabPlan.from_mesh(mesh, cfg.k, cfg.h, cfg.M, cfg.near_radius, world)
        yg = slab.matvec(x)
        assert float((yg - y1).norm() / y1.norm()) <= 1e-13
        slab.close()


@pytest.mark.gpu
def test_slab_nccl_one_rank():
    """The NCCL exchange path (libnccl.so.2 loaded at run time, grouped
    send/recv to self, broadcast) on a one-rank communicator equals the
    single-GPU plan."""
    import torch
    from paper_1712_02443_b200 import AimPlan, AimSlabPlan, nccl_unique_id
    cfg = get_config("c1")
    mesh = make_mesh(cfg)
    single = AimPlan.from_mesh(mesh, cfg.k, cfg.h, cfg.M, cfg.near_radius)
    slab = AimSlabPlan.from_mesh(mesh, cfg.k, cfg.h, cfg.M, cfg.near_radius, 1, 0, nccl_unique_id())
    x = torch.from_numpy(make_vectors(mesh.n_rwg, 3, 5)).cuda()
    y1 = single.matvec(x)
    yg = slab.matvec(x)
    assert float((yg - y1).norm() / y1.norm()) <= 1e-13
    slab.close()
    single.close()


@pytest.mark.gpu
@pytest.mark.parametrize("name,world", [("c1", 3), ("t_m3", 2)])
def test_slab_gmres_matches_single_plan(name, world):
    """aim_slab_gmres (replicated Krylov vectors, distributed products) runs
    the same iteration as aim_gmres on the single plan: equal converged
    counts (+-1) and solutions within the D15 tolerance; the solution's true
    residual checked with an oracle matvec."""
    import torch
    from conftest import oracle_plan
    from oracle.excitation import plane_wave_rhs
    from paper_1712_02443_b200 import AimPlan, AimSlabPlan
    cfg = get_config(name)
    mesh = make_mesh(cfg)
    O = oracle_plan(name)
    V = torch.from_numpy(plane_wave_rhs(O.ctx)).cuda()
    single = AimPlan.from_mesh(mesh, cfg.k, cfg.h, cfg.M, cfg.near_radius)
    slab = AimSlabPlan.from_mesh(mesh, cfg.k, cfg.h, cfg.M, cfg.near_radius, world)
    J1, it1, rr1, st1 = single.gmres(V, restart=50, tol=1e-4)
    Jg, itg, rrg, stg = slab.gmres(V, restart=50, tol=1e-4)
    assert st1 == stg == "AIM_OK" and abs(it1 - itg) <= 1
    assert float((Jg - J1).norm() / J1.norm()) <= 1e-5
    Vh = V.cpu().numpy()
    assert np.linalg.norm(Vh - O.matvec(Jg.cpu().numpy())) / np.linalg.norm(Vh) <= 1e-4 * (1 + 1e-6)
    slab.close()
    single.close()


def _nccl_worker(rank, world, port, name, q):
    """One rank of the multi-process NCCL slab test (one GPU per process)."""
    import torch
    import torch.distributed as dist
    from paper_1712_02443_b200 import AimPlan, AimSlabPlan
    from paper_1712_02443_b200.api import slab_nccl_id
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world)
    cfg = get_config(name)
    mesh = make_mesh(cfg)
    nid = slab_nccl_id()
    slab = AimSlabPlan.from_mesh(mesh, cfg.k, cfg.h, cfg.M, cfg.near_radius, world, rank, nid)
    single = AimPlan.from_mesh(mesh, cfg.k, cfg.h, cfg.M, cfg.near_radius)
    x = torch.from_numpy(make_vectors(mesh.n_rwg, 3, 5)).cuda()
    e_mv = float((slab.matvec(x) - single.matvec(x)).norm() / single.matvec(x).norm())
    V = single.planewave_rhs()
    J1, it1, _, _ = single.gmres(V, restart=50, tol=1e-4)
    Jg, itg, _, st = slab.gmres(V, restart=50, tol=1e-4)
    e_j = float((Jg - J1).norm() / J1.norm())
    q.put((rank, e_mv, it1, itg, st, e_j))
    slab.close()
    single.close()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c1", "t_m3"])
def test_slab_nccl_two_ranks(name):
    """Two processes, one GPU each, NCCL exchanges (halo send/recv, both
    all-to-alls with real peers, the y gather) and the distributed GMRES
    (Krylov vectors split by owner, all-reduced dots): equal to the single
    plan to 1e-13 (product) and +-1 iterations / 1e-5 (GMRES).  Needs two
    GPUs; skipped on a one-GPU box."""
    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_nccl_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, e_mv, it1, itg, st, e_j in res:
        assert e_mv <= 1e-13 and st == "AIM_OK" and abs(it1 - itg) <= 1 and e_j <= 1e-5


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3, 8])
def test_slab_gmres_virtual_worlds_c2(world):
    """The in-process transport walks the NCCL schedule (per-peer offsets of
    both all-to-alls, halos): C2 at full size, G = 2, 3, 8 slabs, the slab
    GMRES on 60 fixed iterations equals the single plan's to 1e-10."""
    import torch
    from paper_1712_02443_b200 import AimPlan, AimSlabPlan
    cfg = get_config("c2")
    mesh = make_mesh(cfg)
    single = AimPlan.from_mesh(mesh, cfg.k, cfg.h, cfg.M, cfg.near_radius)
    V = single.planewave_rhs()
    J1, _, rr1, _ = single.gmres(V, restart=50, tol=1e-4, fixed_iters=60)
    single.close()
    slab = AimSlabPlan.from_mesh(mesh, cfg.k, cfg.h, cfg.M, cfg.near_radius, world)
    Jg, itg, rrg, _ = slab.gmres(V, restart=50, tol=1e-4, fixed_iters=60)
    assert itg == 60
    assert float((Jg - J1).norm() / J1.norm()) <= 1e-10
    assert abs(rrg - rr1) <= 1e-8 * rr1
    slab.close()


@pytest.mark.gpu
@pytest.mark.parametrize("name,world,seq", [("c2", 4, (16, 1, 3)), ("c2", 3, (1,)), ("c4", 2, (1,))])
def test_slab_fused_pack_equals_pack_kernel(name, world, seq, monkeypatch):
    """Planar layouts with a compile-time y plan (C2: 210, C4: 784): the forward
    y pass stores its lines straight into the all-to-all #1 blocks and the
    inverse pass loads them from the received blocks (FftPass::jout / jin).
    Bit-identical to the separate pack / unpack kernels (AIM_SLAB_FUSE_PACK=0),
    2 launches per slab fewer, equal to the single plan to 1e-13; the nrhs
    sequence shrinks below the workspace's nrhs (block offsets scale with nrhs)."""
    import torch
    from paper_1712_02443_b200 import AimPlan, AimSlabPlan, launch_count
    cfg = get_config(name)
    mesh = make_mesh(cfg)
    single = AimPlan.from_mesh(mesh, cfg.k, cfg.h, cfg.M, cfg.near_radius)
    xs = [torch.from_numpy(make_vectors(mesh.n_rwg, r, 11 + r)).cuda() for r in seq]
    y1 = [single.matvec(x) for x in xs]
    single.close()
    slab = AimSlabPlan.from_mesh(mesh, cfg.k, cfg.h, cfg.M, cfg.near_radius, world)
    out = {}
    for fuse in ("1", "0"):
        monkeypatch.setenv("AIM_SLAB_FUSE_PACK", fuse)
        ys, n = [], []
        for x in xs:
            slab.matvec(x)                      # workspace, tables
            c0 = launch_count()
            ys.append(slab.matvec(x))
            n.append(launch_count() - c0)
        out[fuse] = (ys, n)
    for i in range(len(xs)):
        for fuse in ("1", "0"):
            assert float((out[fuse][0][i] - y1[i]).norm() / y1[i].norm()) <= 1e-13, (fuse, i)
        assert torch.equal(out["1"][0][i], out["0"][0][i])
        assert out["0"][1][i] - out["1"][1][i] == 2 * world
    slab.close()
