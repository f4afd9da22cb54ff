"""Python binding with the C-ABI names (argument marshalling only).

Tensors passed in must be contiguous complex128 CUDA tensors on the plan's
device; results are allocated with torch.  The current torch CUDA stream is
passed to the stream-ordered entry points.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

STATUS = {0: "AIM_OK", 1: "AIM_NOT_CONVERGED", -1: "AIM_E_ARG", -2: "AIM_E_MESH", -3: "AIM_E_GRID",
          -4: "AIM_E_NOMEM", -5: "AIM_E_CUDA", -6: "AIM_E_NCCL", -7: "AIM_E_BREAKDOWN"}
C128, C64 = 0, 1   # aim_plan_create precision (AIM_C128, AIM_C64)
EXPORT = {"bases": 0, "weights": 1, "near_rowptr": 2, "near_col": 3, "near_val": 4, "green": 5,
          "proj_rowptr": 6, "proj_ent": 7}


class AimError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def _check(st):
    if st < 0:
        raise AimError(st, _lib.load().aim_last_error().decode())
    return st


def launch_count(reset: bool = False) -> int:
    return int(_lib.load().aim_launch_count(1 if reset else 0))


def _torch():
    import torch
    return torch


def _stream():
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dev_ptr(t, n, nrhs, dtype=None):
    torch = _torch()
    dtype = dtype or torch.complex128
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == dtype and t.is_contiguous()):
        raise TypeError(f"expected a contiguous {dtype} CUDA tensor")
    if t.numel() != n * nrhs:
        raise ValueError(f"expected {n * nrhs} elements, got {t.numel()}")
    return ctypes.c_void_p(t.data_ptr())


class AimPlan:
    """aim_plan_create(...) wrapper; owns the plan until close()."""

    def __init__(self, vertices, triangles, rwg, k, h, M, near_radius, precision=0):
        lib = _lib.load()
        self._v = np.ascontiguousarray(vertices, dtype=np.float64)
        self._t = np.ascontiguousarray(triangles, dtype=np.int32)
        self._r = np.ascontiguousarray(rwg, dtype=np.int32)
        out = ctypes.c_void_p()
        _check(lib.aim_plan_create(self._v.ctypes.data, self._v.shape[0], self._t.ctypes.data, self._t.shape[0],
                                   self._r.ctypes.data, self._r.shape[0], float(k), float(h), int(M),
                                   float(near_radius), int(precision), None, ctypes.byref(out)))
        self._p = out
        self.N = int(self._r.shape[0])
        self.precision = int(precision)
        self.info = self.plan_info()

    @classmethod
    def from_mesh(cls, mesh, k, h, M, near_radius, precision=0):
        return cls(mesh.vertices, mesh.triangles, mesh.rwg, k, h, M, near_radius, precision)

    @property
    def dtype(self):
        """torch dtype of the plan's vectors: complex128 (AIM_C128) or complex64 (AIM_C64)."""
        torch = _torch()
        return torch.complex64 if self.precision == C64 else torch.complex128

    @property
    def np_dtype(self):
        return np.complex64 if self.precision == C64 else np.complex128

    def close(self):
        if getattr(self, "_p", None):
            _lib.load().aim_plan_destroy(self._p)
            self._p = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def plan_info(self) -> dict:
        inf = _lib.AimInfo()
        _check(_lib.load().aim_plan_info(self._p, ctypes.byref(inf)))
        d = {f: getattr(inf, f) for f, _ in _lib.AimInfo._fields_}
        for f in ("grid_origin", "grid_dims", "fft_dims"):
            d[f] = tuple(d[f])
        return d

    @property
    def grid_dims(self):
        return self.info["grid_dims"]

    # ---- hot path
    def matvec(self, x, y=None):
        torch = _torch()
        nrhs = 1 if x.dim() == 1 else x.shape[1]
        if y is None:
            y = torch.empty_like(x)
        _check(_lib.load().aim_matvec(self._p, _dev_ptr(x, self.N, nrhs, self.dtype),
                                      _dev_ptr(y, self.N, nrhs, self.dtype), nrhs, _stream()))
        return y

    def matvec_host(self, x: np.ndarray, y: np.ndarray | None = None) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=self.np_dtype)
        nrhs = 1 if x.ndim == 1 else x.shape[1]
        if y is None:
            y = np.empty_like(x)
        _check(_lib.load().aim_matvec_host(self._p, x.ctypes.data, y.ctypes.data, nrhs))
        return y

    def matvec_host_steps(self, xs, ys):
        """aim_matvec_host_steps: y_i := Z x_i for host arrays (numpy, ideally
        page-locked), copies overlapped with the products inside the library."""
        n = len(xs)
        if len(ys) != n:
            raise ValueError("xs and ys differ in length")
        nrhs = 1 if xs[0].ndim == 1 else xs[0].shape[1]
        for a in list(xs) + list(ys):
            if a.dtype != self.np_dtype or not a.flags.c_contiguous or a.size != self.N * nrhs:
                raise TypeError("host arrays must be contiguous, of the plan's dtype and [N][nrhs]")
        xp = (ctypes.c_void_p * n)(*[a.ctypes.data for a in xs])
        yp = (ctypes.c_void_p * n)(*[a.ctypes.data for a in ys])
        _check(_lib.load().aim_matvec_host_steps(self._p, xp, yp, n, nrhs))
        return ys

    def gmres(self, V, restart=50, tol=1e-4, max_iters=0, fixed_iters=0):
        torch = _torch()
        J = torch.empty_like(V)
        it = ctypes.c_int32()
        rr = ctypes.c_double()
        torch.cuda.current_stream().synchronize()
        st = _check(_lib.load().aim_gmres(self._p, _dev_ptr(V, self.N, 1), _dev_ptr(J, self.N, 1), int(restart),
                                          float(tol), int(max_iters), int(fixed_iters), ctypes.byref(it),
                                          ctypes.byref(rr)))
        return J, int(it.value), float(rr.value), STATUS[st]

    def gmres_history(self) -> np.ndarray:
        """aim_gmres_history: |g_{j+1}|/||V|| of every inner iteration of the last solve."""
        n = ctypes.c_int32()
        _check(_lib.load().aim_gmres_history(self._p, None, 0, ctypes.byref(n)))
        out = np.empty(n.value, dtype=np.float64)
        _check(_lib.load().aim_gmres_history(self._p, out.ctypes.data if out.size else None, out.size,
                                             ctypes.byref(n)))
        return out

    def precond_build(self, kind: int = 1):
        """aim_precond_build: 1 = block-Jacobi over the mesh's connected surfaces, 0 = remove."""
        _check(_lib.load().aim_precond_build(self._p, int(kind)))
        return self.precond_info()

    def precond_info(self) -> dict:
        out = np.zeros(5, dtype=np.int64)
        _check(_lib.load().aim_precond_info(self._p, out.ctypes.data))
        return dict(zip(("built", "elements", "distinct", "max_block", "bytes"), (int(v) for v in out)))

    def precond_apply(self, x):
        torch = _torch()
        y = torch.empty_like(x)
        _check(_lib.load().aim_precond_apply(self._p, _dev_ptr(x, self.N, 1), _dev_ptr(y, self.N, 1), _stream()))
        return y

    # ---- repetition-compressed near field
    def compress(self, mode: int = 1) -> dict:
        """aim_plan_compress: 1 = use the repetition-compressed near field (and, where it pays,
        projection/interpolation templates), 0 = the general tables."""
        _check(_lib.load().aim_plan_compress(self._p, int(mode)))
        return self.compress_info()

    def compress_info(self) -> dict:
        out = np.zeros(6, dtype=np.int64)
        _check(_lib.load().aim_compress_info(self._p, out.ctypes.data))
        return dict(zip(("on", "blocks", "dict_nnz", "nnz_near", "pi_on", "tpl_nnz"), (int(v) for v in out)))

    # ---- array elements and the reduced (macromodel) system
    def elements(self):
        """aim_plan_elements: (element of every RWG [N], translate group of every element)."""
        n = ctypes.c_int32()
        _check(_lib.load().aim_plan_elements(self._p, None, None, ctypes.byref(n)))
        eo = np.empty(self.N, dtype=np.int32)
        gr = np.empty(n.value, dtype=np.int32)
        _check(_lib.load().aim_plan_elements(self._p, eo.ctypes.data, gr.ctypes.data, ctypes.byref(n)))
        return eo, gr

    def reduced_set(self, elem_type, blocks):
        """aim_reduced_set: blocks[d] = (D, T, A, B) complex128 arrays of type d."""
        nhat = np.array([b[0].shape[0] for b in blocks], dtype=np.int32)
        nint = np.array([b[2].shape[0] for b in blocks], dtype=np.int32)
        cat = [np.ascontiguousarray(np.concatenate([np.ascontiguousarray(b[i], dtype=np.complex128).ravel()
                                                    for b in blocks])) for i in range(4)]
        et = np.ascontiguousarray(elem_type, dtype=np.int32)
        _check(_lib.load().aim_reduced_set(self._p, len(blocks), nhat.ctypes.data, nint.ctypes.data,
                                           *[c.ctypes.data for c in cat], et.ctypes.data, et.size))

    def reduced_matvec(self, Y, out=None):
        torch = _torch()
        if out is None:
            out = torch.empty_like(Y)
        _check(_lib.load().aim_reduced_matvec(self._p, _dev_ptr(Y, self.N, 1), _dev_ptr(out, self.N, 1), _stream()))
        return out

    def reduced_gmres(self, V, restart=50, tol=1e-4, max_iters=0, fixed_iters=0):
        torch = _torch()
        E = torch.empty_like(V)
        it = ctypes.c_int32()
        rr = ctypes.c_double()
        torch.cuda.current_stream().synchronize()
        st = _check(_lib.load().aim_reduced_gmres(self._p, _dev_ptr(V, self.N, 1), _dev_ptr(E, self.N, 1),
                                                  int(restart), float(tol), int(max_iters), int(fixed_iters),
                                                  ctypes.byref(it), ctypes.byref(rr)))
        return E, int(it.value), float(rr.value), STATUS[st]

    def planewave_rhs(self, khat=(0.0, 0.0, -1.0), pol=(1.0, 0.0, 0.0), E0=1.0 + 0j):
        torch = _torch()
        V = torch.empty(self.N, dtype=torch.complex128, device="cuda")
        kh = np.ascontiguousarray(khat, dtype=np.float64)
        po = np.ascontiguousarray(pol, dtype=np.float64)
        _check(_lib.load().aim_planewave_rhs(self._p, kh.ctypes.data, po.ctypes.data, float(np.real(E0)),
                                             float(np.imag(E0)), _dev_ptr(V, self.N, 1), _stream()))
        return V

    # ---- stages
    def grid_numel(self, nrhs=1):
        Nx, Ny, Nz = self.grid_dims
        return 4 * Nx * Ny * Nz * nrhs

    def project(self, x):
        torch = _torch()
        nrhs = 1 if x.dim() == 1 else x.shape[1]
        Q = torch.empty(self.grid_numel(nrhs), dtype=self.dtype, device=x.device)
        _check(_lib.load().aim_project(self._p, _dev_ptr(x, self.N, nrhs, self.dtype), ctypes.c_void_p(Q.data_ptr()), nrhs,
                                       _stream()))
        return Q.view(4, *self.grid_dims, nrhs)

    def convolve(self, Q):
        torch = _torch()
        nrhs = Q.shape[-1]
        Phi = torch.empty_like(Q)
        _check(_lib.load().aim_convolve(self._p, ctypes.c_void_p(Q.data_ptr()), ctypes.c_void_p(Phi.data_ptr()),
                                        nrhs, _stream()))
        return Phi

    def interpolate(self, Phi, x=None, add_near=False):
        torch = _torch()
        nrhs = Phi.shape[-1] if Phi is not None else (1 if x.dim() == 1 else x.shape[1])
        y = torch.empty((self.N, nrhs), dtype=self.dtype, device="cuda")
        _check(_lib.load().aim_interpolate(self._p, ctypes.c_void_p(Phi.data_ptr()) if Phi is not None else None,
                                           ctypes.c_void_p(x.data_ptr()) if x is not None else None,
                                           ctypes.c_void_p(y.data_ptr()), nrhs, 1 if add_near else 0, _stream()))
        return y

    # ---- live stage timing
    STAGES = ("project", "fft_x", "fft_yz", "ifft_x", "near_wait", "interp", "near")

    def profile(self, enable: bool):
        _check(_lib.load().aim_profile(self._p, 1 if enable else 0))

    def profile_read(self):
        ms = (ctypes.c_double * 7)()
        cnt = ctypes.c_int64()
        _check(_lib.load().aim_profile_read(self._p, ms, ctypes.byref(cnt)))
        return dict(zip(self.STAGES, list(ms))), int(cnt.value)

    # ---- export
    def export(self, what: str) -> np.ndarray:
        inf = self.info
        N, S = inf["n_rwg"], inf["S"]
        Px, Py, Pz = inf["fft_dims"]
        shapes = {
            "bases": (np.int32, (N, 3)), "weights": (np.float64, (N, S, 4)),
            "near_rowptr": (np.int64, (N + 1,)), "near_col": (np.int32, (inf["nnz_near"],)),
            "near_val": (np.complex128, (inf["nnz_near"],)),
            "green": (np.complex128, (Px // 2 + 1, Py // 2 + 1,
                                      inf["grid_dims"][2] if inf["conv_mode"] != 0 else Pz // 2 + 1)),
            "proj_rowptr": (np.int32, (inf["n_nodes"] + 1,)), "proj_ent": (np.int32, (inf["nnz_proj"],)),
        }
        dt, sh = shapes[what]
        out = np.empty(sh, dtype=dt)
        _check(_lib.load().aim_plan_export(self._p, EXPORT[what], out.ctypes.data, out.nbytes))
        return out


def slab_partition(mesh_or_arrays, h, M, world):
    """aim_slab_partition (host only): slab plane bounds X[world+1], the owning
    rank of every RWG and the grid's x extent Nx."""
    if hasattr(mesh_or_arrays, "vertices"):
        v, t, r = mesh_or_arrays.vertices, mesh_or_arrays.triangles, mesh_or_arrays.rwg
    else:
        v, t, r = mesh_or_arrays
    v = np.ascontiguousarray(v, dtype=np.float64)
    t = np.ascontiguousarray(t, dtype=np.int32)
    r = np.ascontiguousarray(r, dtype=np.int32)
    X = np.empty(world + 1, dtype=np.int32)
    owner = np.empty(r.shape[0], dtype=np.int32)
    nx = ctypes.c_int32()
    _check(_lib.load().aim_slab_partition(v.ctypes.data, v.shape[0], t.ctypes.data, t.shape[0], r.ctypes.data,
                                          r.shape[0], float(h), int(M), int(world), X.ctypes.data,
                                          owner.ctypes.data, ctypes.byref(nx)))
    return X, owner, int(nx.value)


def nccl_unique_id() -> bytes:
    """aim_nccl_unique_id: 128 bytes for aim_slab_create (rank 0 makes it, all ranks use it)."""
    buf = ctypes.create_string_buffer(128)
    _check(_lib.load().aim_nccl_unique_id(buf, 128))
    return buf.raw


class AimSlabPlan:
    """aim_slab_create(...) wrapper: the slab-decomposed operator.
    rank=None: all `world` slabs on the current GPU (device-copy exchanges);
    rank=r with nccl_id: one slab per process/GPU, NCCL exchanges."""

    QUERY = ("X0", "X1", "KY0", "KY1", "n0", "n1", "nnz_near", "a2a_bytes_per_rhs", "halo_bytes_per_rhs", "world")

    def __init__(self, vertices, triangles, rwg, k, h, M, near_radius, world, rank=None, nccl_id=None):
        lib = _lib.load()
        self._v = np.ascontiguousarray(vertices, dtype=np.float64)
        self._t = np.ascontiguousarray(triangles, dtype=np.int32)
        self._r = np.ascontiguousarray(rwg, dtype=np.int32)
        out = ctypes.c_void_p()
        idbuf = ctypes.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        _check(lib.aim_slab_create(self._v.ctypes.data, self._v.shape[0], self._t.ctypes.data, self._t.shape[0],
                                   self._r.ctypes.data, self._r.shape[0], float(k), float(h), int(M),
                                   float(near_radius), int(world), -1 if rank is None else int(rank), idbuf,
                                   ctypes.byref(out)))
        self._p = out
        self.N = int(self._r.shape[0])
        self.world = int(world)
        self.rank = rank

    @classmethod
    def from_mesh(cls, mesh, k, h, M, near_radius, world, rank=None, nccl_id=None):
        return cls(mesh.vertices, mesh.triangles, mesh.rwg, k, h, M, near_radius, world, rank, nccl_id)

    def query(self, rank: int) -> dict:
        out = np.empty(10, dtype=np.int64)
        _check(_lib.load().aim_slab_query(self._p, int(rank), out.ctypes.data))
        return dict(zip(self.QUERY, (int(v) for v in out)))

    def matvec(self, x, y=None):
        torch = _torch()
        nrhs = 1 if x.dim() == 1 else x.shape[1]
        if y is None:
            y = torch.empty_like(x)
        _check(_lib.load().aim_slab_matvec(self._p, _dev_ptr(x, self.N, nrhs), _dev_ptr(y, self.N, nrhs), nrhs,
                                           _stream()))
        return y

    def gmres(self, V, restart=50, tol=1e-4, max_iters=0, fixed_iters=0):
        torch = _torch()
        J = torch.empty_like(V)
        it = ctypes.c_int32()
        rr = ctypes.c_double()
        torch.cuda.current_stream().synchronize()
        st = _check(_lib.load().aim_slab_gmres(self._p, _dev_ptr(V, self.N, 1), _dev_ptr(J, self.N, 1), int(restart),
                                               float(tol), int(max_iters), int(fixed_iters), ctypes.byref(it),
                                               ctypes.byref(rr)))
        return J, int(it.value), float(rr.value), STATUS[st]

    def close(self):
        if getattr(self, "_p", None):
            _lib.load().aim_slab_destroy(self._p)
            self._p = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def slab_nccl_id(group=None) -> bytes:
    """Rank 0 of the torch.distributed group makes an NCCL unique id and every
    rank receives it (host-side plumbing of aim_slab_create with NCCL)."""
    import torch.distributed as dist
    obj = [nccl_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


class HostPipeline:
    """Products from pinned host buffers with the copies overlapped: step i's
    host->device copy, step i-1's product and step i-2's device->host copy run
    on three streams (double-buffered device vectors, event-ordered).  Every
    step still copies its x in and its y out; submit() returns at once, drain()
    waits for everything submitted.  Argument marshalling only: the product is
    aim_matvec on the plan's kernels."""

    def __init__(self, plan: "AimPlan", nrhs: int, depth: int = 2):
        torch = _torch()
        self.plan, self.nrhs, self.depth = plan, nrhs, depth
        shape = (plan.N, nrhs) if nrhs > 1 else (plan.N,)
        self.xd = [torch.empty(shape, dtype=plan.dtype, device="cuda") for _ in range(depth)]
        self.yd = [torch.empty(shape, dtype=plan.dtype, device="cuda") for _ in range(depth)]
        self.s_in, self.s_mv, self.s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
        self.ev_in = [torch.cuda.Event() for _ in range(depth)]
        self.ev_mv = [torch.cuda.Event() for _ in range(depth)]
        self.ev_out = [torch.cuda.Event() for _ in range(depth)]
        self.i = 0

    def submit(self, x_host, y_host):
        """x_host, y_host: pinned torch tensors of the plan's dtype and shape."""
        torch = _torch()
        k = self.i % self.depth
        with torch.cuda.stream(self.s_in):
            if self.i >= self.depth:
                self.s_in.wait_event(self.ev_mv[k])          # slot's x no longer read
            self.xd[k].copy_(x_host, non_blocking=True)
            self.ev_in[k].record(self.s_in)
        with torch.cuda.stream(self.s_mv):
            self.s_mv.wait_event(self.ev_in[k])
            if self.i >= self.depth:
                self.s_mv.wait_event(self.ev_out[k])         # slot's y already copied out
            self.plan.matvec(self.xd[k], self.yd[k])
            self.ev_mv[k].record(self.s_mv)
        with torch.cuda.stream(self.s_out):
            self.s_out.wait_event(self.ev_mv[k])
            y_host.copy_(self.yd[k], non_blocking=True)
            self.ev_out[k].record(self.s_out)
        self.i += 1

    def drain(self):
        for s in (self.s_in, self.s_mv, self.s_out):
            s.synchronize()
