// Slab-decomposed AIM matvec over G ranks (BASELINE.json
// north_star: "the grid is slab-decomposed along x, the 3D FFT transposes run
// as NCCL all-to-all over NVLink, basis functions and precorrection rows are
// partitioned by owning slab with stencil halos").
//
// Partition.  The unpadded grid's x planes are cut into G contiguous slabs
// [X_r, X_{r+1}), balanced by the number of RWGs whose stencil base lies in
// them, every slab at least M planes wide (so a stencil halo only reaches the
// next rank).  Rank r owns those RWGs: their near-field rows, their weights
// and the grid planes [X_r, X_{r+1} + M) their stencils touch.  RWGs are
// renumbered so each rank's rows are contiguous (permuted order = by owner,
// then by id); x is replicated, y is gathered back to every rank.
//
// One product (planar grids, conv_modes 1 and 2; 3-D grids add the z passes):
//   near rows of the owned RWGs (side stream, overlapping everything up to
//     the interpolation) + their projection -> Q on [X_r, X_{r+1} + M)
//   halo reduce: planes [X_{r+1}, X_{r+1} + M) are added into rank r+1
//   y forward FFT (pad Ny -> Py) on the owned planes [3-D: then z forward, pad Nz -> Pz]
//   all-to-all #1: x-slabs -> ky-slabs [KY_s, KY_{s+1}) with every x
//   planar: x forward FFT (pad Nx -> Px), z Toeplitz x G2, x inverse (prune) --
//     mode 1: the fused planar kernel with the roles of x and y swapped
//     (transposed spectrum); mode 2: x pass, z Toeplitz kernel, x pass;
//   3-D: x turnaround (pad, forward, x G^ octant transposed to [ky][kz][kx], inverse, prune)
//   all-to-all #2 back to x-slabs [3-D: z inverse], y inverse FFT (prune Py -> Ny)
//   halo copy: planes [X_{r+1}, X_{r+1} + M) of Phi from rank r+1
//   interpolation of the owned RWGs (accumulates onto the near rows)
//   gather of y (every rank gets all rows), un-permute.
// Every floating-point operation is the single-GPU path's on the same data
// in the same order, except that the projection sums of halo nodes are split
// across two ranks (one extra rounding).
//
// Exchanges run either over NCCL (one process per GPU; libnccl.so.2 loaded at
// run time, grouped send/recv) or, with all G slabs held by one process on one
// GPU, as device copies -- the same packing and offsets, used to check the
// decomposition against the single-GPU plan and the oracle on one device.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <climits>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "aim_internal.cuh"

namespace aim {

static inline unsigned nblk(long long n, int t) { return (unsigned)((n + t - 1) / t); }

// --------------------------------------------------------------- NCCL (dlopen)
struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Bcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    const char* (*ErrStr)(ncclResult_t) = nullptr;
};

static NcclApi& nccl() {
    static NcclApi a;
    if (a.h) return a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw Error(AIM_E_NCCL, std::string("cannot load libnccl.so.2: ") + dlerror());
    auto sym = [&](const char* n) {
        void* f = dlsym(h, n);
        if (!f) throw Error(AIM_E_NCCL, std::string("libnccl.so.2 lacks ") + n);
        return f;
    };
    a.GetUniqueId = (decltype(a.GetUniqueId))sym("ncclGetUniqueId");
    a.CommInitRank = (decltype(a.CommInitRank))sym("ncclCommInitRank");
    a.CommDestroy = (decltype(a.CommDestroy))sym("ncclCommDestroy");
    a.GroupStart = (decltype(a.GroupStart))sym("ncclGroupStart");
    a.GroupEnd = (decltype(a.GroupEnd))sym("ncclGroupEnd");
    a.Send = (decltype(a.Send))sym("ncclSend");
    a.Recv = (decltype(a.Recv))sym("ncclRecv");
    a.Bcast = (decltype(a.Bcast))sym("ncclBroadcast");
    a.AllReduce = (decltype(a.AllReduce))sym("ncclAllReduce");
    a.CommGetAsyncError = (decltype(a.CommGetAsyncError))sym("ncclCommGetAsyncError");
    a.CommAbort = (decltype(a.CommAbort))sym("ncclCommAbort");
    a.ErrStr = (decltype(a.ErrStr))sym("ncclGetErrorString");
    a.h = h;
    return a;
}

#define AIM_NCCL(call)                                                                          \
    do {                                                                                        \
        ncclResult_t r_ = (call);                                                               \
        if (r_ != ncclSuccess) throw Error(AIM_E_NCCL, std::string(#call) + ": " + nccl().ErrStr(r_)); \
    } while (0)

// ------------------------------------------------------------ host partition
// Stencil base x index of every RWG (D3, the same formula as the plan builder)
// and the grid's x extent; then G slabs balanced by RWG count, each >= max(M,1)
// planes.  Host only.
static void slab_partition(const double* V, const int32_t* T, const int32_t* E, int64_t nv, int64_t nt, int64_t N,
                           double h, int M, int G, std::vector<int>& X, std::vector<int>& bx, int& Nx) {
    bx.resize(N);
    long long lo = LLONG_MAX, hi = LLONG_MIN;
    for (int64_t n = 0; n < N; ++n) {
        double cx = 0;
        for (int side = 0; side < 2; ++side) {
            const int32_t t = E[4 * n + 2 + side];
            if (t < 0 || t >= nt) throw Error(AIM_E_MESH, "rwg triangle index out of range");
            for (int c = 0; c < 3; ++c)
                if (T[3 * t + c] < 0 || T[3 * t + c] >= nv) throw Error(AIM_E_MESH, "triangle vertex index out of range");
            cx += (V[3 * T[3 * t]] + V[3 * T[3 * t + 1]] + V[3 * T[3 * t + 2]]) / 3.0;   // as create_plan()
        }
        const double s = floor((0.5 * cx) / h - (M - 1) / 2.0 + 1e-7);
        if (!(fabs(s) < 1e9)) throw Error(AIM_E_GRID, "stencil index exceeds addressable grid");
        bx[n] = (int)s;
        lo = std::min(lo, (long long)s);
        hi = std::max(hi, (long long)s);
    }
    Nx = (int)(hi + M + 1 - lo);
    for (auto& b : bx) b -= (int)lo;
    const int wmin = std::max(M, 1);
    if ((long long)G * wmin > Nx) throw Error(AIM_E_ARG, "more slabs than the grid has x planes for (G * M > Nx)");
    std::vector<long long> cnt(Nx + 1, 0);
    for (int b : bx) cnt[b + 1]++;
    for (int x = 0; x < Nx; ++x) cnt[x + 1] += cnt[x];   // cnt[x] = RWGs with base < x
    X.assign(G + 1, 0);
    X[G] = Nx;
    for (int r = 1; r < G; ++r) {
        const long long target = (long long)r * N / G;
        int x = X[r - 1] + wmin;
        while (x < Nx - (G - r) * wmin && cnt[x] < target) ++x;
        X[r] = std::min(x, Nx - (G - r) * wmin);
    }
}

// ------------------------------------------------------------------ kernels
// y[i] = x[idx[i]] rows of `w` doubles (gather), or y[idx[i]] = x[i] (scatter)
template <bool SCATTER>
__global__ void permute_rows_kernel(const double* __restrict__ x, const int32_t* __restrict__ idx, long long n,
                                    int w, double* __restrict__ y) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n * w) return;
    const long long i = t / w;
    const int c = (int)(t - i * w);
    if (SCATTER) y[(long long)idx[i] * w + c] = x[t];
    else y[t] = x[(long long)idx[i] * w + c];
}

// Near rows of the owned RWGs (permuted ids n0 + i <- global perm[n0 + i]),
// columns renumbered by iperm and re-sorted: the global row is sorted by id,
// the new ids are sorted by (owner, id), so a stable pass per owner value
// restores ascending order.  One thread per row.
__global__ void slab_near_rows_kernel(const int32_t* __restrict__ perm, long long n0, long long nloc,
                                      const int64_t* __restrict__ growp, const int32_t* __restrict__ gcol,
                                      const double2* __restrict__ gval, const int32_t* __restrict__ iperm,
                                      const int32_t* __restrict__ owner, const int64_t* __restrict__ lrowp,
                                      int32_t* __restrict__ lcol, double2* __restrict__ lval, long long N,
                                      long long gnnz, long long* __restrict__ err) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nloc) return;
    const int g = perm[n0 + i];
    if (g < 0 || g >= N) { atomicCAS((unsigned long long*)err, 0ULL, (unsigned long long)(1000000000LL + i)); return; }
    const long long e0 = growp[g], e1 = growp[g + 1];
    if (e0 < 0 || e1 > gnnz || e1 < e0) { atomicCAS((unsigned long long*)err, 0ULL, (unsigned long long)(2000000000LL + i)); return; }
    for (long long e = e0; e < e1; ++e)
        if (gcol[e] < 0 || gcol[e] >= N) { atomicCAS((unsigned long long*)err, 0ULL, (unsigned long long)(3000000000LL + e)); return; }
    if (lrowp[i + 1] - lrowp[i] != e1 - e0) { atomicCAS((unsigned long long*)err, 0ULL, (unsigned long long)(4000000000LL + i)); return; }
    long long o = lrowp[i];
    int cur = -1;
    for (;;) {
        int nxt = INT_MAX;
        for (long long e = e0; e < e1; ++e) {
            const int w = owner[gcol[e]];
            if (w > cur && w < nxt) nxt = w;
        }
        if (nxt == INT_MAX) break;
        for (long long e = e0; e < e1; ++e)
            if (owner[gcol[e]] == nxt) {
                lcol[o] = iperm[gcol[e]];
                lval[o] = gval[e];
                ++o;
            }
        cur = nxt;
    }
}

// spectrum a[AX][AY][AZ] -> planar: b[AY][AX][AZ] (kx <-> ky), 3-D: b[AY][AZ][AX]
template <bool PLANAR>
__global__ void spec_transpose_kernel(const double2* __restrict__ a, int AX, int AY, int AZ, double2* __restrict__ b) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long long)AX * AY * AZ) return;
    const int z = (int)(t % AZ);
    const long long xy = t / AZ;
    const int y = (int)(xy % AY), x = (int)(xy / AY);
    if (PLANAR) b[((long long)y * AX + x) * AZ + z] = a[t];
    else b[((long long)y * AZ + z) * AX + x] = a[t];
}

// All-to-all #1 pack / #2 unpack on rank r:
//   Wy[c][x][ky][zr]  <->  buf[off_s + ((c kys + ky - KY_s) Xl + x) NzR + zr],  s = owner of ky
template <bool UNPACK>
__global__ void slab_pack_kernel(double2* __restrict__ Wy, double2* __restrict__ buf, int Xl, int Py, long long NzR,
                                 const int32_t* __restrict__ kyown, const int32_t* __restrict__ KY,
                                 const long long* __restrict__ off) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long tot = 4LL * Xl * Py * NzR;
    if (t >= tot) return;
    const long long zr = t % NzR;
    long long q = t / NzR;
    const int ky = (int)(q % Py);
    q /= Py;
    const int x = (int)(q % Xl);
    const int c = (int)(q / Xl);
    const int s = kyown[ky];
    const int kys = KY[s + 1] - KY[s];
    const long long b = off[s] + (((long long)c * kys + (ky - KY[s])) * Xl + x) * NzR + zr;
    if (UNPACK) Wy[t] = buf[b];
    else buf[b] = Wy[t];
}

// dst[i] += src[i]
__global__ void add_kernel(double2* __restrict__ dst, const double2* __restrict__ src, long long n) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        const double2 a = dst[i], b = src[i];
        dst[i] = make_double2(a.x + b.x, a.y + b.y);
    }
}

}  // namespace aim

// ------------------------------------------------------------------ plan
struct aim_slab_rank {
    int rank = 0;
    int X0 = 0, X1 = 0, Xl = 0, Xh = 0;   // owned planes [X0, X1), with halo [X0, X0 + Xh)
    int KY0 = 0, KY1 = 0;                 // owned ky range of the x-pencil phase
    int64_t n0 = 0, n1 = 0;               // permuted row range
    aim_plan* sub = nullptr;              // local tables (N = n1 - n0, grid Xh x Ny x Nz)
    // workspaces (complex128), sized for ws_nrhs
    double2* Qh = nullptr;    // [4][Xh][Ny][Nz][R]   projection (+halo) / Phi (+halo)
    double2* Wy = nullptr;    // [4][Xl][Py][Zc][R]   after the y (3-D: and z) forward pass
    double2* Wy1 = nullptr;   // [4][Xl][Py][Nz][R]   3-D only: between the y and z passes
    double2* T = nullptr;     // [4][KYl][Nx][Zc][R]  x pencils
    double2* Tp = nullptr;    // [4][KYl][Px][Nz][R]  conv mode 2: x-padded pencils
    double2* sb = nullptr;    // send blocks  (max of the two all-to-alls)
    double2* rb = nullptr;    // receive blocks
    double2* hb = nullptr;    // halo staging [4][M][Ny][Nz][R]
    long long* d_off1 = nullptr;   // pack offsets of all-to-all #1, per destination
    long long* d_jtab = nullptr;   // [4][Py] planar: element offset of line (c, ky) in the packed blocks
                                   // (the pack fused into the y-pass store, the unpack into its load)
};

struct aim_slab {
    int world = 1, rank = -1;             // rank < 0: all slabs in this process
    bool virt = true;
    aim_plan* base = nullptr;             // full single-GPU plan (spectrum, FFT axes, grid dims)
    int Nx = 0, Ny = 0, Nz = 0, Px = 0, Py = 0, Pz = 0, M = 0;
    int planar = 1;
    int Zc = 0;                           // z extent of the exchanged layout: Nz (planar) or Pz (3-D)
    int64_t N = 0;
    std::vector<int> X, KY;
    std::vector<int64_t> nstart;
    std::vector<aim_slab_rank> ranks;     // all (virtual) or the own one
    int32_t* perm = nullptr;              // [N] permuted row -> RWG id
    int32_t* kyown = nullptr;             // [Py] owner of ky
    int32_t* d_KY = nullptr;              // [world+1]
    double2* g2t = nullptr;               // transposed spectrum (planar [ay][ax][dz], 3-D [ay][az][ax])
    double2* xp = nullptr;                // [N][R] permuted x
    double2* yp = nullptr;                // [N][R] permuted y
    int ws_nrhs = 0;
    int tab_nrhs = 0;                      // nrhs the offset tables (d_off1, d_jtab) were written for
    ncclComm_t comm = nullptr;
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;          // near-field rows, overlapping the FFT and its all-to-alls
    cudaEvent_t ev_x = nullptr, ev_n = nullptr;
    std::vector<std::pair<void*, size_t>> allocs;
    int64_t bytes_a2a = 0, bytes_halo = 0;   // per matvec and RHS, per rank (max)
    double2* gm_b = nullptr;              // distributed GMRES: local right-hand side / solution
    double2* gm_x = nullptr;
    long long gm_n = 0;

    template <class T>
    T* alloc(size_t n) {
        void* p = nullptr;
        if (n == 0) n = 1;
        const cudaError_t e = cudaMalloc(&p, n * sizeof(T));
        if (e != cudaSuccess) throw aim::Error(AIM_E_NOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
        allocs.emplace_back(p, n * sizeof(T));
        return (T*)p;
    }
    void release(void* p) {
        if (!p) return;
        for (size_t i = 0; i < allocs.size(); ++i)
            if (allocs[i].first == p) {
                allocs.erase(allocs.begin() + i);
                break;
            }
        cudaFree(p);
    }
};

namespace aim {

static int owner_of(const std::vector<int>& X, int bx) {
    return (int)(std::upper_bound(X.begin(), X.end(), bx) - X.begin()) - 1;
}

static void slab_destroy(aim_slab* S) {
    if (!S) return;
    cudaDeviceSynchronize();
    for (auto& R : S->ranks)
        if (R.sub) destroy_plan(R.sub);
    if (S->base) destroy_plan(S->base);
    for (auto& a : S->allocs) cudaFree(a.first);
    if (S->comm) nccl().CommDestroy(S->comm);
    if (S->stream) cudaStreamDestroy(S->stream);
    if (S->side) cudaStreamDestroy(S->side);
    if (S->ev_x) cudaEventDestroy(S->ev_x);
    if (S->ev_n) cudaEventDestroy(S->ev_n);
    delete S;
}

static void slab_create(const double* V, int64_t nv, const int32_t* T, int64_t nt, const int32_t* E, int64_t N,
                        double k, double h, int M, double r, int world, int rank, const void* nccl_id, aim_slab* S) {
    S->world = world;
    S->rank = rank;
    S->virt = rank < 0;
    S->N = N;
    S->M = M;
    AIM_CUDA(cudaStreamCreateWithFlags(&S->stream, cudaStreamNonBlocking));
    AIM_CUDA(cudaStreamCreateWithFlags(&S->side, cudaStreamNonBlocking));
    AIM_CUDA(cudaEventCreateWithFlags(&S->ev_x, cudaEventDisableTiming));
    AIM_CUDA(cudaEventCreateWithFlags(&S->ev_n, cudaEventDisableTiming));
    cudaStream_t s = S->stream;
    // partition (host formula, checked below against the plan's own stencil bases)
    std::vector<int> bx;
    int Nx = 0;
    slab_partition(V, T, E, nv, nt, N, h, M, world, S->X, bx, Nx);
    // base plan: the grid, weights, projection and spectrum of the whole
    // operator; with one rank per process the near rows (the dominant plan
    // time and memory) only for the RWGs this rank owns
    S->base = new aim_plan();
    if (!S->virt) {
        S->base->near_keep.resize(N);
        for (int64_t n = 0; n < N; ++n) S->base->near_keep[n] = owner_of(S->X, bx[n]) == rank;
    }
    create_plan(V, nv, T, nt, E, N, k, h, M, r, AIM_C128, S->base);
    aim_plan* B = S->base;
    S->planar = B->planar;
    if (S->planar == 1 && !planar_supported(B->pads[0], B->dims[2], B->ax[0].min_radix))
        throw Error(AIM_E_ARG, "planar slab pass: the x lines do not fit the planar kernel");
    S->Nx = B->dims[0]; S->Ny = B->dims[1]; S->Nz = B->dims[2];
    S->Px = B->pads[0]; S->Py = B->pads[1]; S->Pz = B->pads[2];
    S->Zc = S->planar ? S->Nz : S->Pz;
    if (Nx != S->Nx) throw Error(AIM_E_GRID, "slab partition disagrees with the plan's grid");
    std::vector<int32_t> pb(3 * N);
    AIM_CUDA(cudaMemcpy(pb.data(), B->base, sizeof(int32_t) * 3 * N, cudaMemcpyDeviceToHost));
    std::vector<int32_t> owner(N), perm, iperm(N);
    for (int64_t n = 0; n < N; ++n) {
        if (pb[3 * n] - B->origin[0] != bx[n]) throw Error(AIM_E_GRID, "slab partition: stencil base mismatch");
        owner[n] = owner_of(S->X, bx[n]);
    }
    perm.reserve(N);
    S->nstart.assign(world + 1, 0);
    for (int w = 0; w < world; ++w) {
        for (int64_t n = 0; n < N; ++n)
            if (owner[n] == w) perm.push_back((int32_t)n);
        S->nstart[w + 1] = (int64_t)perm.size();
    }
    for (int64_t i = 0; i < N; ++i) iperm[perm[i]] = (int32_t)i;
    S->KY.assign(world + 1, 0);
    for (int w = 0; w <= world; ++w) S->KY[w] = (int)((long long)w * S->Py / world);
    std::vector<int32_t> kyown(S->Py);
    for (int w = 0; w < world; ++w)
        for (int ky = S->KY[w]; ky < S->KY[w + 1]; ++ky) kyown[ky] = w;
    auto up = [&](const std::vector<int32_t>& v) {
        int32_t* d = S->alloc<int32_t>(v.size());
        h2d(d, v.data(), sizeof(int32_t) * v.size(), s);
        return d;
    };
    S->perm = up(perm);
    S->kyown = up(kyown);
    S->d_KY = up(std::vector<int32_t>(S->KY.begin(), S->KY.end()));
    int32_t* d_iperm = up(iperm);
    int32_t* d_owner = up(owner);
    // transposed spectrum for the x-pencil pass
    const int AX = S->Px / 2 + 1, AY = S->Py / 2 + 1, AZ = S->planar ? S->Nz : S->Pz / 2 + 1;
    S->g2t = S->alloc<double2>((size_t)AX * AY * AZ);
    if (S->planar)
        spec_transpose_kernel<true><<<nblk((long long)AX * AY * AZ, 256), 256, 0, s>>>(B->spec, AX, AY, AZ, S->g2t);
    else
        spec_transpose_kernel<false><<<nblk((long long)AX * AY * AZ, 256), 256, 0, s>>>(B->spec, AX, AY, AZ, S->g2t);
    note_launch("slab_spec_transpose");
    std::vector<int64_t> growp(N + 1);
    AIM_CUDA(cudaMemcpy(growp.data(), B->nrow, sizeof(int64_t) * (N + 1), cudaMemcpyDeviceToHost));

    // local tables of every rank this process holds
    for (int w = 0; w < world; ++w) {
        if (!S->virt && w != rank) continue;
        aim_slab_rank R;
        R.rank = w;
        R.X0 = S->X[w];
        R.X1 = S->X[w + 1];
        R.Xl = R.X1 - R.X0;
        R.Xh = std::min(R.Xl + M, S->Nx - R.X0);
        R.KY0 = S->KY[w];
        R.KY1 = S->KY[w + 1];
        R.n0 = S->nstart[w];
        R.n1 = S->nstart[w + 1];
        const long long nl = R.n1 - R.n0;
        aim_plan* q = new aim_plan();
        R.sub = q;
        q->device = B->device;
        q->N = nl; q->nt = B->nt; q->nv = B->nv; q->k = k; q->h = h; q->M = M; q->r = r; q->S = B->S;
        q->prec = AIM_C128;
        q->planar = 1;
        q->dims[0] = R.Xh; q->dims[1] = S->Ny; q->dims[2] = S->Nz;
        for (int d = 0; d < 3; ++d) q->pads[d] = B->pads[d];
        q->origin[0] = B->origin[0] + R.X0; q->origin[1] = B->origin[1]; q->origin[2] = B->origin[2];
        q->Ng = (long long)R.Xh * S->Ny * S->Nz;
        // rows of the owned RWGs: centres, weights, grid bases (local)
        const int32_t* dperm = S->perm + R.n0;
        q->rwg_c = q->alloc<double>(3 * std::max<long long>(nl, 1));
        q->W = q->alloc<double>((size_t)std::max<long long>(nl, 1) * q->S * 4);
        if (nl) {
            permute_rows_kernel<false><<<nblk(nl * 3, 256), 256, 0, s>>>(B->rwg_c, dperm, nl, 3, q->rwg_c);
            permute_rows_kernel<false><<<nblk(nl * q->S * 4, 256), 256, 0, s>>>(B->W, dperm, nl, q->S * 4, q->W);
            note_launch("slab_rows");
        }
        std::vector<int32_t> node0(nl);
        for (long long i = 0; i < nl; ++i) {
            const int64_t g = perm[R.n0 + i];
            const int lx = pb[3 * g] - B->origin[0] - R.X0, ly = pb[3 * g + 1] - B->origin[1],
                      lz = pb[3 * g + 2] - B->origin[2];
            node0[i] = (int32_t)(((long long)lx * S->Ny + ly) * S->Nz + lz);
        }
        q->node0 = q->alloc<int32_t>(std::max<long long>(nl, 1));
        if (nl) h2d(q->node0, node0.data(), sizeof(int32_t) * nl, s);
        build_projection_csr(q, node0, s);
        // near rows: columns renumbered and re-sorted
        std::vector<int64_t> lrowp(nl + 1, 0);
        for (long long i = 0; i < nl; ++i) {
            const int64_t g = perm[R.n0 + i];
            lrowp[i + 1] = lrowp[i] + (growp[g + 1] - growp[g]);
        }
        q->nnzN = lrowp[nl];
        q->nrow = q->alloc<int64_t>(nl + 3);
        q->ncol = q->alloc<int32_t>(q->nnzN + 4);
        q->nval = q->alloc<double2>(q->nnzN + 1);
        q->ncol_padded = 1;
        h2d(q->nrow, lrowp.data(), sizeof(int64_t) * (nl + 1), s);
        // AIM_SLAB_RANK_NEAR=1 (tests): with all slabs in one process, take each
        // rank's near rows from its own base plan built with that rank's
        // near_keep, as a one-rank-per-process rank does (the owned rows'
        // lists are the same; the others are empty)
        aim_plan* NB = B;
        const char* rn = getenv("AIM_SLAB_RANK_NEAR");
        if (S->virt && rn && rn[0] == '1') {
            NB = new aim_plan();
            NB->near_keep.resize(N);
            for (int64_t n = 0; n < N; ++n) NB->near_keep[n] = owner[n] == w;
            try {
                create_plan(V, nv, T, nt, E, N, k, h, M, r, AIM_C128, NB);
            } catch (...) {
                destroy_plan(NB);
                throw;
            }
        }
        struct NbGuard {
            aim_plan* nb; aim_plan* b;
            ~NbGuard() { if (nb != b) destroy_plan(nb); }
        } nb_guard{NB, B};
        if (nl) {
            long long* d_err = nullptr;
            AIM_CUDA(cudaMalloc(&d_err, sizeof(long long)));
            AIM_CUDA(cudaMemsetAsync(d_err, 0, sizeof(long long), s));
            slab_near_rows_kernel<<<nblk(nl, 128), 128, 0, s>>>(S->perm, R.n0, nl, NB->nrow, NB->ncol, NB->nval,
                                                                d_iperm, d_owner, q->nrow, q->ncol, q->nval, N,
                                                                NB->nnzN, d_err);
            note_launch("slab_near_rows");
            long long herr = 0;
            AIM_CUDA(cudaMemcpyAsync(&herr, d_err, sizeof(long long), cudaMemcpyDeviceToHost, s));
            AIM_CUDA(cudaStreamSynchronize(s));
            cudaFree(d_err);
            if (herr)
                throw Error(AIM_E_GRID, "slab near rows: bad index code " + std::to_string(herr) + " rank " +
                                            std::to_string(w) + " nl " + std::to_string(nl) + " nnz " +
                                            std::to_string(q->nnzN) + " gnnz " + std::to_string(NB->nnzN));
        }
        AIM_CUDA(cudaStreamSynchronize(s));
        S->ranks.push_back(R);
    }
    S->release(d_iperm);
    S->release(d_owner);
    // the full plan's per-RWG tables are no longer needed
    for (void* ptr : {(void*)B->W, (void*)B->nval, (void*)B->ncol, (void*)B->pent, (void*)B->prow, (void*)B->pn,
                      (void*)B->Wc})
        B->release(ptr);
    B->W = nullptr; B->nval = nullptr; B->ncol = nullptr; B->pent = nullptr; B->prow = nullptr; B->pn = nullptr;
    B->Wc = nullptr;
    if (!S->virt) {
        if (!nccl_id) throw Error(AIM_E_ARG, "rank >= 0 needs an NCCL unique id");
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, sizeof(id));
        AIM_NCCL(nccl().CommInitRank(&S->comm, world, id, rank));
    }
    // exchange volume per RHS (max over ranks): all-to-all out + in, halos
    for (int w = 0; w < world; ++w) {
        const long long Xl = S->X[w + 1] - S->X[w], kys = S->KY[w + 1] - S->KY[w];
        const long long out = 4 * Xl * (S->Py - kys) * S->Zc * 16, in = 4 * kys * (S->Nx - Xl) * S->Zc * 16;
        S->bytes_a2a = std::max<int64_t>(S->bytes_a2a, 2 * (out + in));
    }
    S->bytes_halo = 2LL * 4 * M * S->Ny * S->Nz * 16 * (world > 1 ? 2 : 0);
}

// Offsets of the all-to-all #1 blocks for exactly R right-hand sides (they scale
// with R, so a product with fewer RHS than the workspace was sized for needs its own).
static void slab_tables(aim_slab* S, int R) {
    if (S->tab_nrhs == R) return;
    // products of the previous nrhs may still be reading the tables on the caller's stream
    AIM_CUDA(cudaDeviceSynchronize());
    const long long ZR = (long long)S->Zc * R;
    for (auto& Rk : S->ranks) {
        std::vector<long long> off(S->world + 1, 0);
        for (int w = 0; w < S->world; ++w) off[w + 1] = off[w] + 4LL * (S->KY[w + 1] - S->KY[w]) * Rk.Xl * ZR;
        h2d(Rk.d_off1, off.data(), sizeof(long long) * (S->world + 1), S->stream);
        // line (c, ky) of the y-transformed slab starts at off[s] + ((c kys + ky - KY_s) Xl) ZR, s = owner of ky
        std::vector<long long> jt(4 * (size_t)S->Py);
        for (int c = 0; c < 4; ++c)
            for (int w = 0; w < S->world; ++w) {
                const long long kys = S->KY[w + 1] - S->KY[w];
                for (int ky = S->KY[w]; ky < S->KY[w + 1]; ++ky)
                    jt[(size_t)c * S->Py + ky] = off[w] + ((c * kys + (ky - S->KY[w])) * Rk.Xl) * ZR;
            }
        h2d(Rk.d_jtab, jt.data(), sizeof(long long) * jt.size(), S->stream);
    }
    S->tab_nrhs = R;
}

static void slab_workspace(aim_slab* S, int R) {
    if (S->ws_nrhs >= R) {
        slab_tables(S, R);
        return;
    }
    AIM_CUDA(cudaDeviceSynchronize());
    S->release(S->xp);
    S->release(S->yp);
    S->xp = S->alloc<double2>((size_t)S->N * R);
    S->yp = S->alloc<double2>((size_t)S->N * R);
    const long long NzR = (long long)S->Nz * R, ZR = (long long)S->Zc * R;
    for (auto& Rk : S->ranks) {
        for (void* ptr : {(void*)Rk.Qh, (void*)Rk.Wy, (void*)Rk.Wy1, (void*)Rk.T, (void*)Rk.Tp, (void*)Rk.sb,
                          (void*)Rk.rb, (void*)Rk.hb, (void*)Rk.d_off1, (void*)Rk.d_jtab})
            S->release(ptr);
        Rk.Wy1 = nullptr;
        Rk.Tp = nullptr;
        const long long kyl = Rk.KY1 - Rk.KY0;
        Rk.Qh = S->alloc<double2>(4LL * Rk.Xh * S->Ny * NzR);
        Rk.Wy = S->alloc<double2>(4LL * Rk.Xl * S->Py * ZR);
        if (!S->planar) Rk.Wy1 = S->alloc<double2>(4LL * Rk.Xl * S->Py * NzR);
        Rk.T = S->alloc<double2>(4LL * kyl * S->Nx * ZR);
        if (S->planar == 2) Rk.Tp = S->alloc<double2>(4LL * kyl * S->Px * ZR);
        const long long blk = std::max(4LL * Rk.Xl * S->Py * ZR, 4LL * kyl * S->Nx * ZR);
        Rk.sb = S->alloc<double2>(blk);
        Rk.rb = S->alloc<double2>(blk);
        Rk.hb = S->alloc<double2>(4LL * S->M * S->Ny * NzR);
        Rk.d_off1 = S->alloc<long long>(S->world + 1);
        Rk.d_jtab = S->alloc<long long>(4 * (size_t)S->Py);
    }
    S->ws_nrhs = R;
    S->tab_nrhs = 0;
    slab_tables(S, R);
}

static aim_slab_rank* rank_of(aim_slab* S, int w) {
    for (auto& R : S->ranks)
        if (R.rank == w) return &R;
    return nullptr;
}

// The all-to-all pack fused into the y-pass store (and the unpack into the
// inverse pass's load): planar layouts only (the y pass is the last before the
// exchange), AIM_SLAB_FUSE_PACK=0 keeps the separate pack kernel.
static bool slab_fuse_pack(const aim_slab* S) {
    const char* e = getenv("AIM_SLAB_FUSE_PACK");
    return S->planar && !(e && e[0] == '0');
}

// one y pass per component: [Xl][Ny -> Py][NzR] forward (Qh -> Y) or
// [Xl][Py -> Ny][NzR] inverse (Y -> Qh); Y = Wy (planar) or Wy1 (3-D).
// With `xbuf` (planar, fused exchange layout) the forward pass writes its lines
// straight into the all-to-all #1 blocks of xbuf and the inverse pass reads them
// from there (d_jtab); returns false if no table-addressed kernel takes the
// pass (nothing launched: the caller runs the plain pass and the pack kernel).
static bool slab_ypass(aim_slab* S, aim_slab_rank& Rk, int R, bool inverse, cudaStream_t s, double2* xbuf = nullptr) {
    const long long NzR = (long long)S->Nz * R;
    double2* Y = S->planar ? Rk.Wy : Rk.Wy1;
    for (int c = 0; c < 4; ++c) {
        FftPass f{};
        f.prec = AIM_C128;
        f.outer = Rk.Xl;
        f.inner = NzR;
        f.ax = S->base->ax[1];
        f.TO = f.TI = 0;
        if (!inverse) {
            f.in = Rk.Qh + c * (long long)Rk.Xh * S->Ny * NzR;
            f.out = Y + c * (long long)Rk.Xl * S->Py * NzR;
            f.Lin = S->Ny; f.Lout = S->Py; f.mode = 0;
            if (xbuf) { f.out = xbuf; f.jout = Rk.d_jtab + (size_t)c * S->Py; }
        } else {
            f.in = Y + c * (long long)Rk.Xl * S->Py * NzR;
            f.out = Rk.Qh + c * (long long)Rk.Xh * S->Ny * NzR;
            f.Lin = S->Py; f.Lout = S->Ny; f.mode = 1;
            if (xbuf) { f.in = xbuf; f.jin = Rk.d_jtab + (size_t)c * S->Py; }
        }
        if (xbuf) {
            if (!try_launch_fft_pass_tab(f, s)) {
                if (c) throw Error(AIM_E_GRID, "slab y pass: table-addressed kernel refused component " + std::to_string(c));
                return false;
            }
        } else {
            launch_fft_pass(f, s);
        }
    }
    return true;
}

// 3-D only: z pass over [4 Xl Py][Nz -> Pz][R] (Wy1 -> Wy) or back (Wy -> Wy1)
static void slab_zpass(aim_slab* S, aim_slab_rank& Rk, int R, bool inverse, cudaStream_t s) {
    FftPass f{};
    f.prec = AIM_C128;
    f.outer = 4LL * Rk.Xl * S->Py;
    f.inner = R;
    f.ax = S->base->ax[2];
    f.TO = f.TI = 0;
    f.in = inverse ? Rk.Wy : Rk.Wy1;
    f.out = inverse ? Rk.Wy1 : Rk.Wy;
    f.Lin = inverse ? S->Pz : S->Nz;
    f.Lout = inverse ? S->Nz : S->Pz;
    f.mode = inverse ? 1 : 0;
    launch_fft_pass(f, s);
}

// halo planes [Xl, Xh) of every component, packed [4][Xh - Xl][Ny][NzR]
static void halo_copy(aim_slab* S, const aim_slab_rank& Rk, double2* grid, double2* buf, bool to_buf, int first,
                      int planes, int R, cudaStream_t s) {
    const size_t plane = sizeof(double2) * (size_t)S->Ny * S->Nz * R;
    for (int c = 0; c < 4; ++c) {
        char* g = (char*)(grid + (size_t)c * Rk.Xh * S->Ny * S->Nz * R) + plane * first;
        char* b = (char*)buf + plane * planes * c;
        if (to_buf) AIM_CUDA(cudaMemcpyAsync(b, g, plane * planes, cudaMemcpyDeviceToDevice, s));
        else AIM_CUDA(cudaMemcpyAsync(g, b, plane * planes, cudaMemcpyDeviceToDevice, s));
    }
}

static void check_nccl(aim_slab* S);

// Point-to-point exchanges of one phase: every rank this
// process holds posts its sends and receives, then run() executes them --
// over NCCL (one rank per process: grouped ncclSend/ncclRecv, then an async
// error check that aborts the communicator so peers do not hang), or, with
// all ranks in this process, as device copies matching each receive with the
// send posted for it.  Both modes walk the same schedule, buffers and offsets.
struct Transport {
    aim_slab* S;
    cudaStream_t s;
    struct Op {
        int self, peer;
        double2* buf;
        size_t n;   // doubles
    };
    std::vector<Op> sends, recvs;
    void send(int self, const double2* buf, size_t n, int to) { sends.push_back({self, to, (double2*)buf, n}); }
    void recv(int self, double2* buf, size_t n, int from) { recvs.push_back({self, from, buf, n}); }
    void run() {
        if (!S->virt) {
            NcclApi& nc = nccl();
            AIM_NCCL(nc.GroupStart());
            for (size_t i = 0; i < std::max(sends.size(), recvs.size()); ++i) {
                if (i < sends.size() && sends[i].n)
                    AIM_NCCL(nc.Send(sends[i].buf, sends[i].n, ncclDouble, sends[i].peer, S->comm, s));
                if (i < recvs.size() && recvs[i].n)
                    AIM_NCCL(nc.Recv(recvs[i].buf, recvs[i].n, ncclDouble, recvs[i].peer, S->comm, s));
            }
            AIM_NCCL(nc.GroupEnd());
            check_nccl(S);
        } else {
            std::vector<char> used(sends.size(), 0);
            for (const Op& r : recvs) {
                size_t k = 0;
                while (k < sends.size() && (used[k] || sends[k].self != r.peer || sends[k].peer != r.self)) ++k;
                if (k == sends.size() || sends[k].n != r.n)
                    throw Error(AIM_E_ARG, "slab exchange: receive " + std::to_string(r.peer) + " -> " +
                                               std::to_string(r.self) + " has no matching send");
                used[k] = 1;
                if (r.n)
                    AIM_CUDA(cudaMemcpyAsync(r.buf, sends[k].buf, sizeof(double) * r.n, cudaMemcpyDeviceToDevice, s));
            }
            for (char u : used)
                if (!u) throw Error(AIM_E_ARG, "slab exchange: a send without a matching receive");
        }
        sends.clear();
        recvs.clear();
    }
};

// After NCCL work is enqueued: a failed or timed-out peer shows up as an
// asynchronous error; abort the communicator so the other ranks do not hang.
static void check_nccl(aim_slab* S) {
    if (S->virt || !S->comm) return;
    ncclResult_t st = ncclSuccess;
    AIM_NCCL(nccl().CommGetAsyncError(S->comm, &st));
    if (st != ncclSuccess && st != ncclInProgress) {
        nccl().CommAbort(S->comm);
        S->comm = nullptr;
        throw Error(AIM_E_NCCL, std::string("NCCL asynchronous error: ") + nccl().ErrStr(st));
    }
}

// The slab product on permuted, replicated x (S->xp): rows [n0, n1) of every
// held rank are written to S->yp.
static void slab_core(aim_slab* S, int R, cudaStream_t s) {
    const int G = S->world, M = S->M;
    const long long NzR = (long long)S->Nz * R, ZR = (long long)S->Zc * R;
    const size_t esz = sizeof(double2);
    Transport T{S, s, {}, {}};
    // near rows on the side stream (they overlap the projection, the FFT passes
    // and the all-to-alls; interpolation waits for them), projection on `s`
    AIM_CUDA(cudaEventRecord(S->ev_x, s));
    AIM_CUDA(cudaStreamWaitEvent(S->side, S->ev_x, 0));
    for (auto& Rk : S->ranks)
        if (Rk.n1 > Rk.n0) launch_near(Rk.sub, S->xp, S->yp + Rk.n0 * R, R, S->side);
    AIM_CUDA(cudaEventRecord(S->ev_n, S->side));
    for (auto& Rk : S->ranks) {
        if (Rk.n1 > Rk.n0) {
            launch_project(Rk.sub, S->xp + Rk.n0 * R, Rk.Qh, R, s);
        } else {
            AIM_CUDA(cudaMemsetAsync(Rk.Qh, 0, esz * 4 * Rk.Xh * S->Ny * NzR, s));
        }
    }
    // halo reduce: planes [Xl, Xl + M) of rank w are added into planes [0, M)
    // of rank w+1 (every slab is >= M planes wide; the last has no halo)
    const size_t hcnt = 2 * (size_t)4 * M * S->Ny * NzR;   // doubles
    for (auto& Rk : S->ranks) {
        const int w = Rk.rank;
        if (w + 1 < G) {
            halo_copy(S, Rk, Rk.Qh, Rk.hb, true, Rk.Xl, M, R, s);
            T.send(w, Rk.hb, hcnt, w + 1);
        }
        if (w > 0) T.recv(w, Rk.rb, hcnt, w - 1);
    }
    T.run();
    for (auto& Rk : S->ranks) {
        if (Rk.rank == 0) continue;
        halo_copy(S, Rk, Rk.Qh, Rk.sb, true, 0, M, R, s);
        add_kernel<<<nblk(hcnt / 2, 256), 256, 0, s>>>(Rk.sb, Rk.rb, (long long)(hcnt / 2));
        note_launch("slab_halo_add");
        halo_copy(S, Rk, Rk.Qh, Rk.sb, false, 0, M, R, s);
    }
    // y (3-D: and z) forward on the owned planes, pack for all-to-all #1
    for (auto& Rk : S->ranks) {
        if (slab_fuse_pack(S) && slab_ypass(S, Rk, R, false, s, Rk.sb)) continue;   // lines stored into the blocks
        slab_ypass(S, Rk, R, false, s);
        if (!S->planar) slab_zpass(S, Rk, R, false, s);
        const long long tot = 4LL * Rk.Xl * S->Py * ZR;
        slab_pack_kernel<false><<<nblk(tot, 256), 256, 0, s>>>(Rk.Wy, Rk.sb, Rk.Xl, S->Py, ZR, S->kyown, S->d_KY,
                                                                Rk.d_off1);
        note_launch("slab_pack");
    }
    // all-to-all #1: block (w -> v) = [4 kys_v][Xl_w][ZR] at sb(w) offset off1(w, v);
    // rank v receives the blocks of w = 0 .. G-1 back to back in rb and places
    // each at x = X_w of its pencils T
    auto blk1 = [&](int w, int v) { return 4LL * (S->KY[v + 1] - S->KY[v]) * (S->X[w + 1] - S->X[w]) * ZR; };
    auto off1 = [&](int w, int v) {
        long long o = 0;
        for (int u = 0; u < v; ++u) o += blk1(w, u);
        return o;
    };
    auto offr = [&](int v, int w) {   // receive offset of the block from w on rank v
        long long o = 0;
        for (int u = 0; u < w; ++u) o += blk1(u, v);
        return o;
    };
    auto place = [&](aim_slab_rank& Dv, const double2* src, int w, bool into_T) {
        // rows (c, kyl) of width Xl_w ZR: T_v[c][kyl][X_w + x][zr] <-> src[c][kyl][x][zr]
        const long long Xl = S->X[w + 1] - S->X[w], kys = Dv.KY1 - Dv.KY0;
        const size_t wb = esz * Xl * ZR, tp = esz * (size_t)S->Nx * ZR;
        char* t = (char*)(Dv.T + (long long)S->X[w] * ZR);
        if (into_T) AIM_CUDA(cudaMemcpy2DAsync(t, tp, src, wb, wb, 4 * kys, cudaMemcpyDeviceToDevice, s));
        else AIM_CUDA(cudaMemcpy2DAsync((void*)src, wb, t, tp, wb, 4 * kys, cudaMemcpyDeviceToDevice, s));
    };
    for (auto& Rk : S->ranks) {
        const int w = Rk.rank;
        for (int v = 0; v < G; ++v) {
            T.send(w, Rk.sb + off1(w, v), 2 * (size_t)blk1(w, v), v);
            T.recv(w, Rk.rb + offr(w, v), 2 * (size_t)blk1(v, w), v);
        }
    }
    T.run();
    for (auto& Rk : S->ranks)
        for (int v = 0; v < G; ++v) place(Rk, Rk.rb + offr(Rk.rank, v), v, true);
    // x forward, z Toeplitz x G2 (3-D: x G^), x inverse on the ky pencils
    for (auto& Rk : S->ranks) {
        if (S->planar == 2) {
            // separate passes: x forward (pad) into Tp, z Toeplitz (ky = KY0 + a, kx = b), x inverse (prune)
            const int kyl = Rk.KY1 - Rk.KY0;
            if (kyl <= 0) continue;
            FftPass f{};
            f.prec = AIM_C128;
            f.outer = 4LL * kyl;
            f.inner = ZR;
            f.ax = S->base->ax[0];
            f.TO = f.TI = 0;
            f.in = Rk.T; f.out = Rk.Tp; f.Lin = S->Nx; f.Lout = S->Px; f.mode = 0;
            launch_fft_pass(f, s);
            launch_ztoeplitz(Rk.Tp, AIM_C128, kyl, S->Px, S->Nz, R, 0, Rk.KY0, S->Px, S->Py, S->base->spec, s);
            f.TO = f.TI = 0;
            f.in = Rk.Tp; f.out = Rk.T; f.Lin = S->Px; f.Lout = S->Nx; f.mode = 1;
            launch_fft_pass(f, s);
            continue;
        }
        if (!S->planar) {
            FftPass f{};
            f.prec = AIM_C128;
            f.in = Rk.T;
            f.out = Rk.T;
            f.outer = 4LL * (Rk.KY1 - Rk.KY0);
            f.Lin = f.Lout = S->Nx;
            f.inner = ZR;
            f.mode = 2;
            f.ax = S->base->ax[0];
            f.TO = f.TI = 0;
            f.spec = S->g2t;
            f.spec_mode = 1;
            f.Px = S->Px; f.Py = S->Py; f.Pz = S->Pz;
            f.PxH = S->Px / 2 + 1; f.PyH = S->Py / 2 + 1; f.PzH = S->Pz / 2 + 1;
            f.off = Rk.KY0; f.nky = std::max(1, Rk.KY1 - Rk.KY0); f.Rin = R;
            if (f.outer > 0) launch_fft_pass(f, s);
            continue;
        }
        PlanarPass q{};
        q.prec = AIM_C128;
        q.W = Rk.T;
        q.Px = Rk.KY1 - Rk.KY0;
        q.Ny = S->Nx;
        q.Nz = S->Nz;
        q.R = R;
        q.PyH = S->Px / 2 + 1;
        q.ay = S->base->ax[0];
        q.spec = S->g2t;
        q.off = Rk.KY0;
        q.Pfold = S->Py;
        if (q.Px > 0) launch_planar_yz(q, s);
    }
    // all-to-all #2 (reverse): rank v packs its pencil rows at x = X_w back to
    // back in sb (offset offr(v, w)) and sends them to w, which receives them at
    // rb offset off1(w, v) -- the layout all-to-all #1 read from -- and unpacks
    for (auto& Rk : S->ranks)
        for (int w = 0; w < G; ++w) place(Rk, Rk.sb + offr(Rk.rank, w), w, false);
    for (auto& Rk : S->ranks) {
        const int v = Rk.rank;
        for (int w = 0; w < G; ++w) {
            T.send(v, Rk.sb + offr(v, w), 2 * (size_t)blk1(w, v), w);
            T.recv(v, Rk.rb + off1(v, w), 2 * (size_t)blk1(v, w), w);
        }
    }
    T.run();
    for (auto& Rk : S->ranks) {
        if (slab_fuse_pack(S) && slab_ypass(S, Rk, R, true, s, Rk.rb)) continue;    // lines loaded from the blocks
        const long long tot = 4LL * Rk.Xl * S->Py * ZR;
        slab_pack_kernel<true><<<nblk(tot, 256), 256, 0, s>>>(Rk.Wy, Rk.rb, Rk.Xl, S->Py, ZR, S->kyown, S->d_KY,
                                                               Rk.d_off1);
        note_launch("slab_unpack");
        if (!S->planar) slab_zpass(S, Rk, R, true, s);
        slab_ypass(S, Rk, R, true, s);   // Phi on the owned planes, into Qh
    }
    // Phi halo: planes [Xl, Xl + M) of rank w <- planes [0, M) of rank w+1
    for (auto& Rk : S->ranks) {
        const int w = Rk.rank;
        if (w > 0) {
            halo_copy(S, Rk, Rk.Qh, Rk.rb, true, 0, M, R, s);
            T.send(w, Rk.rb, hcnt, w - 1);
        }
        if (w + 1 < G) T.recv(w, Rk.hb, hcnt, w + 1);
    }
    T.run();
    for (auto& Rk : S->ranks)
        if (Rk.rank + 1 < G) halo_copy(S, Rk, Rk.Qh, Rk.hb, false, Rk.Xl, M, R, s);
    // interpolation of the owned RWGs onto their near rows
    AIM_CUDA(cudaStreamWaitEvent(s, S->ev_n, 0));
    for (auto& Rk : S->ranks)
        if (Rk.n1 > Rk.n0) launch_interp(Rk.sub, Rk.Qh, S->yp + Rk.n0 * R, R, true, s);
}

// every rank receives all rows of a permuted row vector (NCCL: a broadcast
// from each owner; in-process the ranks share the vector already)
static void slab_allgather_rows(aim_slab* S, double2* v, int R, cudaStream_t s) {
    if (S->virt) return;
    NcclApi& nc = nccl();
    AIM_NCCL(nc.GroupStart());
    for (int w = 0; w < S->world; ++w) {
        double2* blk = v + S->nstart[w] * R;
        const size_t cnt = 2 * (size_t)(S->nstart[w + 1] - S->nstart[w]) * R;
        if (cnt) AIM_NCCL(nc.Bcast(blk, blk, cnt, ncclDouble, w, S->comm, s));
    }
    AIM_NCCL(nc.GroupEnd());
    check_nccl(S);
}

static void slab_matvec(aim_slab* S, const double2* x, double2* y, int R, cudaStream_t s) {
    slab_workspace(S, R);
    const long long N = S->N;
    permute_rows_kernel<false><<<nblk(N * 2 * R, 256), 256, 0, s>>>((const double*)x, S->perm, N, 2 * R,
                                                                     (double*)S->xp);
    note_launch("slab_permute");
    slab_core(S, R, s);
    slab_allgather_rows(S, S->yp, R, s);
    permute_rows_kernel<true><<<nblk(N * 2 * R, 256), 256, 0, s>>>((const double*)S->yp, S->perm, N, 2 * R,
                                                                    (double*)y);
    note_launch("slab_unpermute");
}

// GMRES on the slab operator (D15) with the Krylov vectors partitioned by
// owning rank: each rank keeps its rows [n0, n1) of the
// permuted order; a product gathers the rank's rows of its input into every
// rank's x (one broadcast per owner), runs the slab product and keeps its
// own rows; dot products are local partial sums followed by an NCCL
// all-reduce of the (j+1) coefficients.  In-process (all ranks held) the
// vectors span all rows and no reduction is needed.
static int slab_gmres(aim_slab* S, const double2* V, double2* J, int restart, double tol, int max_iters,
                      int fixed_iters, int* iters, double* rel_res) {
    cudaStream_t s = S->base->stream;
    slab_workspace(S, 1);
    const long long N = S->N;
    const long long n0 = S->virt ? 0 : S->ranks[0].n0;
    const long long nl = S->virt ? N : S->ranks[0].n1 - S->ranks[0].n0;
    // permuted right-hand side, local rows
    permute_rows_kernel<false><<<nblk(N * 2, 256), 256, 0, s>>>((const double*)V, S->perm, N, 2, (double*)S->yp);
    note_launch("slab_permute");
    if (S->gm_n < nl) {
        S->release(S->gm_b);
        S->release(S->gm_x);
        S->gm_b = S->alloc<double2>(std::max<long long>(1, nl));
        S->gm_x = S->alloc<double2>(std::max<long long>(1, nl));
        S->gm_n = nl;
    }
    AIM_CUDA(cudaMemcpyAsync(S->gm_b, S->yp + n0, sizeof(double2) * nl, cudaMemcpyDeviceToDevice, s));
    GmresOps ops;
    ops.n = nl;
    ops.matvec = [S, n0, nl](const double2* in, double2* out, cudaStream_t st) {
        AIM_CUDA(cudaMemcpyAsync(S->xp + n0, in, sizeof(double2) * nl, cudaMemcpyDeviceToDevice, st));
        slab_allgather_rows(S, S->xp, 1, st);
        slab_core(S, 1, st);
        AIM_CUDA(cudaMemcpyAsync(out, S->yp + n0, sizeof(double2) * nl, cudaMemcpyDeviceToDevice, st));
    };
    if (!S->virt)
        ops.allreduce = [S](double2* d, int n, cudaStream_t st) {
            AIM_NCCL(nccl().AllReduce(d, d, 2 * (size_t)n, ncclDouble, ncclSum, S->comm, st));
            check_nccl(S);
        };
    const int st = gmres_core(S->base, ops, S->gm_b, S->gm_x, restart, tol, max_iters, fixed_iters, iters, rel_res);
    // J replicated in the caller's order
    AIM_CUDA(cudaMemcpyAsync(S->yp + n0, S->gm_x, sizeof(double2) * nl, cudaMemcpyDeviceToDevice, s));
    slab_allgather_rows(S, S->yp, 1, s);
    permute_rows_kernel<true><<<nblk(N * 2, 256), 256, 0, s>>>((const double*)S->yp, S->perm, N, 2, (double*)J);
    note_launch("slab_unpermute");
    AIM_CUDA(cudaStreamSynchronize(s));
    return st;
}

}  // namespace aim

using namespace aim;

extern "C" {

int aim_slab_partition(const double* vertices, int64_t nv, const int32_t* triangles, int64_t nt,
                       const int32_t* rwg_edges, int64_t n_rwg, double h, int32_t M, int32_t world, int32_t* X,
                       int32_t* owner, int32_t* grid_nx) {
    if (!vertices || !triangles || !rwg_edges || !X || n_rwg < 1 || world < 1 || !(h > 0) || M < 1 || M > 6)
        return fail(AIM_E_ARG, "bad argument");
    return guarded([&] {
        std::vector<int> Xv, bx;
        int Nx = 0;
        slab_partition(vertices, triangles, rwg_edges, nv, nt, n_rwg, h, M, world, Xv, bx, Nx);
        for (int w = 0; w <= world; ++w) X[w] = Xv[w];
        if (owner)
            for (int64_t n = 0; n < n_rwg; ++n) owner[n] = owner_of(Xv, bx[n]);
        if (grid_nx) *grid_nx = Nx;
        return AIM_OK;
    });
}

int aim_nccl_unique_id(void* id, int64_t bytes) {
    if (!id || bytes != (int64_t)sizeof(ncclUniqueId)) return fail(AIM_E_ARG, "id buffer must be NCCL_UNIQUE_ID_BYTES");
    return guarded([&] {
        ncclUniqueId u;
        AIM_NCCL(nccl().GetUniqueId(&u));
        std::memcpy(id, &u, sizeof(u));
        return AIM_OK;
    });
}

int aim_slab_create(const double* vertices, int64_t nv, const int32_t* triangles, int64_t nt,
                    const int32_t* rwg_edges, int64_t n_rwg, double k, double h, int32_t M, double near_radius,
                    int32_t world, int32_t rank, const void* nccl_id, aim_slab** out) {
    if (!out) return fail(AIM_E_ARG, "out is NULL");
    *out = nullptr;
    if (!vertices || !triangles || !rwg_edges || n_rwg < 1 || world < 1 || rank >= world)
        return fail(AIM_E_ARG, "bad argument");
    if (!(k > 0) || !(h > 0) || M < 1 || M > 6 || !(near_radius >= 0))
        return fail(AIM_E_ARG, "k, h > 0, M in [1,6], near_radius >= 0 required");
    aim_slab* S = new aim_slab();
    const int st = guarded([&] {
        slab_create(vertices, nv, triangles, nt, rwg_edges, n_rwg, k, h, M, near_radius, world, rank, nccl_id, S);
        return AIM_OK;
    });
    if (st != AIM_OK) {
        const std::string msg = last_error();
        slab_destroy(S);
        last_error() = msg;
        return st;
    }
    *out = S;
    return AIM_OK;
}

// A rank that fails after its peers entered a collective would leave them
// blocked: abort the communicator on any error of a collective entry point.
static int abort_on_error(aim_slab* S, int st) {
    if (st < 0 && S && !S->virt && S->comm) {
        nccl().CommAbort(S->comm);
        S->comm = nullptr;
    }
    return st;
}

int aim_slab_matvec(aim_slab* S, const void* x, void* y, int32_t nrhs, void* stream) {
    if (!S || !x || !y || nrhs < 1 || x == y) return fail(AIM_E_ARG, "bad argument");
    if (!S->virt && !S->comm) return fail(AIM_E_NCCL, "the communicator was aborted after an earlier error");
    return abort_on_error(S, guarded([&] {
        slab_matvec(S, (const double2*)x, (double2*)y, nrhs, (cudaStream_t)stream);
        return AIM_OK;
    }));
}

int aim_slab_gmres(aim_slab* S, const void* V, void* J, int32_t restart, double tol, int32_t max_iters,
                   int32_t fixed_iters, int32_t* iters, double* rel_res) {
    if (!S || !V || !J || restart < 1 || !(tol >= 0)) return fail(AIM_E_ARG, "bad argument");
    if (!S->virt && !S->comm) return fail(AIM_E_NCCL, "the communicator was aborted after an earlier error");
    return abort_on_error(S, guarded([&] {
        int it = 0;
        double rr = 0;
        const int st = slab_gmres(S, (const double2*)V, (double2*)J, restart, tol, max_iters, fixed_iters, &it, &rr);
        if (iters) *iters = it;
        if (rel_res) *rel_res = rr;
        return st;
    }));
}

int aim_slab_query(const aim_slab* S, int32_t rank, int64_t* out) {
    if (!S || !out || rank < 0 || rank >= S->world) return fail(AIM_E_ARG, "bad argument");
    return guarded([&] {
        out[0] = S->X[rank];
        out[1] = S->X[rank + 1];
        out[2] = S->KY[rank];
        out[3] = S->KY[rank + 1];
        out[4] = S->nstart[rank];
        out[5] = S->nstart[rank + 1];
        const aim_slab_rank* R = nullptr;
        for (auto& r : S->ranks)
            if (r.rank == rank) R = &r;
        out[6] = R ? R->sub->nnzN : -1;
        out[7] = S->bytes_a2a;
        out[8] = S->bytes_halo;
        out[9] = S->world;
        return AIM_OK;
    });
}

int aim_slab_destroy(aim_slab* S) {
    return guarded([&] {
        slab_destroy(S);
        return AIM_OK;
    });
}

}  // extern "C"
