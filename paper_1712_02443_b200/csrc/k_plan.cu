// Plan construction on the device (setup steps S2-S4 of SURVEY.md §8(a)):
//   S2 projection weights (tensor Lagrange moment matching, D2) and the
//      grid-node-sorted projection CSR (deterministic, no atomics);
//   S3 Green's-function spectrum (sampled min-image kernel, forward FFT via
//      the same Stockham passes as the matvec, octant storage, D11/D12);
//   S4 near list (cell list, ||c_m - c_n|| <= r(1+1e-9), D5), exact Galerkin
//      EFIE entries with singularity subtraction (D8), symmetrisation (D9) and
//      precorrection Z_corr = Z_ex_sym - Z_grid.
#include <math.h>

#include <algorithm>
#include <cstdlib>
#include <climits>
#include <numeric>
#include <vector>

#include "aim_internal.cuh"

namespace aim {

static inline unsigned nblk(long long n, int t) { return (unsigned)((n + t - 1) / t); }
static inline unsigned nblk_of(long long n) { return (unsigned)((n + 127) / 128); }

// ------------------------------------------------------------ S2 weights
// L_i(t) = prod_{j != i} (t - j)/(i - j) on nodes 0..M
template <int M>
__device__ __forceinline__ double lagr(double t, int i) {
    double num = 1.0, den = 1.0;
#pragma unroll
    for (int j = 0; j <= M; ++j)
        if (j != i) {
            num *= (t - j);
            den *= (double)(i - j);
        }
    return num / den;
}

template <int M>
__global__ void weights_kernel(const double* __restrict__ qp, const double* __restrict__ qw,
                               const int32_t* __restrict__ rt, const double* __restrict__ ra,
                               const double* __restrict__ rp, const int32_t* __restrict__ base, double h,
                               long long N, double* __restrict__ W) {
    constexpr int M1 = M + 1, S = M1 * M1 * M1;
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= N * S) return;
    const long long n = idx / S;
    const int u = (int)(idx % S);
    const int i = u / (M1 * M1), j = (u / M1) % M1, kk = u % M1;
    const double bx = base[3 * n], by = base[3 * n + 1], bz = base[3 * n + 2];
    double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
    for (int side = 0; side < 2; ++side) {
        const int t = rt[2 * n + side];
        const double a = ra[2 * n + side];
        const double px = rp[6 * n + 3 * side], py = rp[6 * n + 3 * side + 1], pz = rp[6 * n + 3 * side + 2];
        for (int q = 0; q < 7; ++q) {
            const double x = qp[(7 * t + q) * 3], y = qp[(7 * t + q) * 3 + 1], z = qp[(7 * t + q) * 3 + 2];
            const double L = lagr<M>(x / h - bx, i) * lagr<M>(y / h - by, j) * lagr<M>(z / h - bz, kk);
            const double f = qw[7 * t + q] * L;
            acc0 += f * a * (x - px);
            acc1 += f * a * (y - py);
            acc2 += f * a * (z - pz);
            acc3 += f * 2.0 * a;
        }
    }
    double2* o = reinterpret_cast<double2*>(W + 4 * idx);
    o[0] = make_double2(acc0, acc1);
    o[1] = make_double2(acc2, acc3);
}

void build_weights(aim_plan* p, cudaStream_t s) {
    p->W = p->alloc<double>((size_t)p->N * p->S * 4);
    const long long tot = p->N * p->S;
    switch (p->M) {
#define W_CASE(MM) \
    case MM: weights_kernel<MM><<<nblk(tot, 256), 256, 0, s>>>(p->tri_qp, p->tri_qw, p->rwg_t, p->rwg_a, p->rwg_p, p->base, p->h, p->N, p->W); break;
        W_CASE(1) W_CASE(2) W_CASE(3) W_CASE(4) W_CASE(5) W_CASE(6)
#undef W_CASE
    }
    note_launch("weights");
}

// ------------------------------------------------- S2 projection CSR (nodes)
// Entries of node g: for u (ascending), for n in bucket(g - o_u) (ascending):
// ent = n*S + u.  bucket(b) = RWGs whose stencil base node is b.
__global__ void proj_count_kernel(const int32_t* __restrict__ bptr, int Nx, int Ny, int Nz, int M,
                                  int32_t* __restrict__ cnt) {
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long Ng = (long long)Nx * Ny * Nz;
    if (g >= Ng) return;
    const int x = (int)(g / ((long long)Ny * Nz)), y = (int)((g / Nz) % Ny), z = (int)(g % Nz);
    int c = 0;
    for (int i = 0; i <= M; ++i)
        for (int j = 0; j <= M; ++j)
            for (int k = 0; k <= M; ++k) {
                const int bx = x - i, by = y - j, bz = z - k;
                if (bx < 0 || by < 0 || bz < 0) continue;
                const long long b = ((long long)bx * Ny + by) * Nz + bz;
                c += bptr[b + 1] - bptr[b];
            }
    cnt[g] = c;
}

__global__ void proj_fill_kernel(const int32_t* __restrict__ bptr, const int32_t* __restrict__ bids, int Nx,
                                 int Ny, int Nz, int M, const int32_t* __restrict__ prow,
                                 int32_t* __restrict__ pent) {
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long Ng = (long long)Nx * Ny * Nz;
    if (g >= Ng) return;
    const int M1 = M + 1, S = M1 * M1 * M1;
    const int x = (int)(g / ((long long)Ny * Nz)), y = (int)((g / Nz) % Ny), z = (int)(g % Nz);
    int pos = prow[g];
    for (int i = 0; i <= M; ++i)
        for (int j = 0; j <= M; ++j)
            for (int k = 0; k <= M; ++k) {
                const int bx = x - i, by = y - j, bz = z - k;
                if (bx < 0 || by < 0 || bz < 0) continue;
                const long long b = ((long long)bx * Ny + by) * Nz + bz;
                const int u = (i * M1 + j) * M1 + k;
                for (int e = bptr[b]; e < bptr[b + 1]; ++e) pent[pos++] = bids[e] * S + u;
            }
}

// pn[e] = n, Wc[e][0..3] = W[n][u][0..3] for entry e = n S + u
__global__ void proj_gather_kernel(const int32_t* __restrict__ pent, long long nnz, int S,
                                   const double* __restrict__ W, int32_t* __restrict__ pn, double* __restrict__ Wc) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nnz) return;
    const int ent = pent[e];
    pn[e] = ent / S;
    const double2* src = reinterpret_cast<const double2*>(W) + 2 * (long long)ent;
    double2* dst = reinterpret_cast<double2*>(Wc) + 2 * e;
    dst[0] = src[0];
    dst[1] = src[1];
}

void build_projection_csr(aim_plan* p, const std::vector<int32_t>& node0, cudaStream_t s) {
    const long long Ng = p->Ng;
    // counting sort of RWGs by base node (stable: ascending n inside a bucket)
    std::vector<int32_t> bptr(Ng + 1, 0), bids(p->N);
    for (long long n = 0; n < p->N; ++n) bptr[node0[n] + 1]++;
    for (long long g = 0; g < Ng; ++g) bptr[g + 1] += bptr[g];
    {
        std::vector<int32_t> fill(bptr.begin(), bptr.end() - 1);
        for (long long n = 0; n < p->N; ++n) bids[fill[node0[n]]++] = (int32_t)n;
    }
    int32_t* d_bptr = nullptr;
    int32_t* d_bids = nullptr;
    int32_t* d_cnt = nullptr;
    AIM_CUDA(cudaMalloc(&d_bptr, sizeof(int32_t) * (Ng + 1)));
    AIM_CUDA(cudaMalloc(&d_bids, sizeof(int32_t) * std::max<long long>(1, p->N)));
    AIM_CUDA(cudaMalloc(&d_cnt, sizeof(int32_t) * Ng));
    AIM_CUDA(cudaMemcpyAsync(d_bptr, bptr.data(), sizeof(int32_t) * (Ng + 1), cudaMemcpyHostToDevice, s));
    AIM_CUDA(cudaMemcpyAsync(d_bids, bids.data(), sizeof(int32_t) * p->N, cudaMemcpyHostToDevice, s));
    proj_count_kernel<<<nblk(Ng, 256), 256, 0, s>>>(d_bptr, p->dims[0], p->dims[1], p->dims[2], p->M, d_cnt);
    note_launch("proj_count");
    std::vector<int32_t> cnt(Ng);
    AIM_CUDA(cudaMemcpyAsync(cnt.data(), d_cnt, sizeof(int32_t) * Ng, cudaMemcpyDeviceToHost, s));
    AIM_CUDA(cudaStreamSynchronize(s));
    std::vector<int32_t> prow(Ng + 1, 0);
    long long acc = 0;
    for (long long g = 0; g < Ng; ++g) {
        prow[g] = (int32_t)acc;
        acc += cnt[g];
    }
    prow[Ng] = (int32_t)acc;
    if (acc != p->N * p->S) throw Error(AIM_E_GRID, "projection CSR count mismatch");
    p->nnzP = acc;
    p->prow = p->alloc<int32_t>(Ng + 1);
    p->pent = p->alloc<int32_t>(acc);
    AIM_CUDA(cudaMemcpyAsync(p->prow, prow.data(), sizeof(int32_t) * (Ng + 1), cudaMemcpyHostToDevice, s));
    proj_fill_kernel<<<nblk(Ng, 256), 256, 0, s>>>(d_bptr, d_bids, p->dims[0], p->dims[1], p->dims[2], p->M,
                                                   p->prow, p->pent);
    note_launch("proj_fill");
    // the weights in CSR order (projection streams them instead of gathering)
    p->pn = p->alloc<int32_t>(acc);
    p->Wc = p->alloc<double>(4 * (size_t)std::max<long long>(acc, 1));
    if (acc) {
        proj_gather_kernel<<<nblk(acc, 256), 256, 0, s>>>(p->pent, acc, p->S, p->W, p->pn, p->Wc);
        note_launch("proj_gather");
    }
    AIM_CUDA(cudaStreamSynchronize(s));
    cudaFree(d_bptr);
    cudaFree(d_bids);
    cudaFree(d_cnt);
}

// ------------------------------------------------------------- S4 near list
struct CellGrid {
    double lo[3];
    double csz;
    int nc[3];
    int32_t* cptr;  // [ncells+1]
    int32_t* cids;  // [N]
};

__device__ __forceinline__ bool near_pair(const double* c, long long m, long long n, double lim) {
    const double dx = __dsub_rn(c[3 * m], c[3 * n]);
    const double dy = __dsub_rn(c[3 * m + 1], c[3 * n + 1]);
    const double dz = __dsub_rn(c[3 * m + 2], c[3 * n + 2]);
    const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
    return __dsqrt_rn(d2) <= lim;
}

__device__ __forceinline__ int cell_of(double v, double lo, double csz, int nc) {
    int c = (int)floor((v - lo) / csz);
    return min(max(c, 0), nc - 1);
}

template <bool FILL>
__global__ void near_scan_kernel(const double* __restrict__ cen, long long N, CellGrid cg, double lim,
                                 const int64_t* __restrict__ rowp, int32_t* __restrict__ out_cnt,
                                 int32_t* __restrict__ out_col) {
    const long long m = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= N) return;
    int cx = cell_of(cen[3 * m], cg.lo[0], cg.csz, cg.nc[0]);
    int cy = cell_of(cen[3 * m + 1], cg.lo[1], cg.csz, cg.nc[1]);
    int cz = cell_of(cen[3 * m + 2], cg.lo[2], cg.csz, cg.nc[2]);
    if (FILL && rowp[m + 1] == rowp[m]) return;   // a row dropped by near_keep (every kept row holds m itself)
    long long pos = FILL ? rowp[m] : 0;
    int cnt = 0;
    for (int ax = max(cx - 1, 0); ax <= min(cx + 1, cg.nc[0] - 1); ++ax)
        for (int ay = max(cy - 1, 0); ay <= min(cy + 1, cg.nc[1] - 1); ++ay)
            for (int az = max(cz - 1, 0); az <= min(cz + 1, cg.nc[2] - 1); ++az) {
                const long long cell = ((long long)ax * cg.nc[1] + ay) * cg.nc[2] + az;
                for (int e = cg.cptr[cell]; e < cg.cptr[cell + 1]; ++e) {
                    const int n = cg.cids[e];
                    if (near_pair(cen, m, n, lim)) {
                        if (FILL) out_col[pos++] = n;
                        else ++cnt;
                    }
                }
            }
    if (!FILL) out_cnt[m] = cnt;
}

// warp per row: rank sort (columns are distinct) tmp -> col
__global__ void near_sort_kernel(const int64_t* __restrict__ rowp, long long N, const int32_t* __restrict__ tmp,
                                 int32_t* __restrict__ col) {
    const long long m = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / 32;
    const int lane = threadIdx.x & 31;
    if (m >= N) return;
    const long long a = rowp[m], b = rowp[m + 1];
    for (long long e = a + lane; e < b; e += 32) {
        const int v = tmp[e];
        int rank = 0;
        for (long long f = a; f < b; ++f) rank += (tmp[f] < v);
        col[a + rank] = v;
    }
}

void build_near_list(aim_plan* p, cudaStream_t s) {
    const long long N = p->N;
    std::vector<double> cen(3 * N);
    AIM_CUDA(cudaMemcpy(cen.data(), p->rwg_c, sizeof(double) * 3 * N, cudaMemcpyDeviceToHost));
    const double lim = p->r * (1.0 + 1e-9);
    double lo[3], hi[3];
    for (int a = 0; a < 3; ++a) {
        lo[a] = 1e300;
        hi[a] = -1e300;
    }
    for (long long n = 0; n < N; ++n)
        for (int a = 0; a < 3; ++a) {
            lo[a] = std::min(lo[a], cen[3 * n + a]);
            hi[a] = std::max(hi[a], cen[3 * n + a]);
        }
    double ext = std::max({hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2], 1e-30});
    CellGrid cg;
    cg.csz = std::max(lim * 1.01, ext / 256.0);
    long long ncells = 1;
    for (int a = 0; a < 3; ++a) {
        cg.lo[a] = lo[a];
        cg.nc[a] = (int)std::floor((hi[a] - lo[a]) / cg.csz) + 1;
        ncells *= cg.nc[a];
    }
    std::vector<int32_t> cell(N), cptr(ncells + 1, 0), cids(N);
    for (long long n = 0; n < N; ++n) {
        int c[3];
        for (int a = 0; a < 3; ++a)
            c[a] = std::min(std::max((int)std::floor((cen[3 * n + a] - cg.lo[a]) / cg.csz), 0), cg.nc[a] - 1);
        cell[n] = (int32_t)(((long long)c[0] * cg.nc[1] + c[1]) * cg.nc[2] + c[2]);
        cptr[cell[n] + 1]++;
    }
    for (long long c = 0; c < ncells; ++c) cptr[c + 1] += cptr[c];
    {
        std::vector<int32_t> f(cptr.begin(), cptr.end() - 1);
        for (long long n = 0; n < N; ++n) cids[f[cell[n]]++] = (int32_t)n;
    }
    AIM_CUDA(cudaMalloc(&cg.cptr, sizeof(int32_t) * (ncells + 1)));
    AIM_CUDA(cudaMalloc(&cg.cids, sizeof(int32_t) * N));
    h2d(cg.cptr, cptr.data(), sizeof(int32_t) * (ncells + 1), s);
    h2d(cg.cids, cids.data(), sizeof(int32_t) * N, s);
    int32_t* d_cnt = nullptr;
    AIM_CUDA(cudaMalloc(&d_cnt, sizeof(int32_t) * N));
    near_scan_kernel<false><<<nblk(N, 256), 256, 0, s>>>(p->rwg_c, N, cg, lim, nullptr, d_cnt, nullptr);
    note_launch("near_count");
    std::vector<int32_t> cnt(N);
    AIM_CUDA(cudaMemcpyAsync(cnt.data(), d_cnt, sizeof(int32_t) * N, cudaMemcpyDeviceToHost, s));
    AIM_CUDA(cudaStreamSynchronize(s));
    // rows a slab rank does not own get no near entries (aim_plan::near_keep)
    if (!p->near_keep.empty())
        for (long long m = 0; m < N; ++m)
            if (!p->near_keep[m]) cnt[m] = 0;
    std::vector<int64_t> rowp(N + 1, 0);
    for (long long m = 0; m < N; ++m) rowp[m + 1] = rowp[m] + cnt[m];
    const long long nnz = rowp[N];
    if (nnz > 2147483647LL) throw Error(AIM_E_GRID, "near-field nnz exceeds 2^31-1");
    p->nnzN = nnz;
    p->nrow = p->alloc<int64_t>(N + 3);   // + bulk-copy slack
    p->ncol = p->alloc<int32_t>(nnz + 4);  // + bulk-copy slack (k_near_stream.cu)
    AIM_CUDA(cudaMemcpyAsync(p->nrow, rowp.data(), sizeof(int64_t) * (N + 1), cudaMemcpyHostToDevice, s));
    int32_t* tmp = nullptr;
    AIM_CUDA(cudaMalloc(&tmp, sizeof(int32_t) * std::max<long long>(1, nnz)));
    near_scan_kernel<true><<<nblk(N, 256), 256, 0, s>>>(p->rwg_c, N, cg, lim, p->nrow, nullptr, tmp);
    note_launch("near_fill");
    near_sort_kernel<<<nblk(N * 32, 256), 256, 0, s>>>(p->nrow, N, tmp, p->ncol);
    note_launch("near_sort");
    AIM_CUDA(cudaStreamSynchronize(s));
    cudaFree(tmp);
    cudaFree(d_cnt);
    cudaFree(cg.cptr);
    cudaFree(cg.cids);
}

// ------------------------------------------------- near field, 4-row blocks
// Union of the (sorted) column lists of the block's rows, by a 4-way merge;
// FILL writes the columns and the dense 4-value groups (0 where a row lacks
// the column).  One thread per block.
template <bool FILL>
__global__ void near_block_kernel(const int32_t* __restrict__ rows, long long nblk, const int64_t* __restrict__ rowp,
                                  const int32_t* __restrict__ col, const double2* __restrict__ val,
                                  const int64_t* __restrict__ bptr, int64_t* __restrict__ bcnt,
                                  int32_t* __restrict__ bcol, double2* __restrict__ bval) {
    const long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nblk) return;
    long long pos[4], end[4];
    for (int i = 0; i < 4; ++i) {
        const int r = rows[4 * b + i];
        pos[i] = r >= 0 ? rowp[r] : 0;
        end[i] = r >= 0 ? rowp[r + 1] : 0;
    }
    long long out = FILL ? bptr[b] : 0;
    long long cnt = 0;
    for (;;) {
        int c = INT_MAX;
        for (int i = 0; i < 4; ++i)
            if (pos[i] < end[i]) c = min(c, col[pos[i]]);
        if (c == INT_MAX) break;
        double2 v[4];
        for (int i = 0; i < 4; ++i) {
            v[i] = make_double2(0.0, 0.0);
            if (pos[i] < end[i] && col[pos[i]] == c) {
                if (FILL) v[i] = val[pos[i]];
                ++pos[i];
            }
        }
        if (FILL) {
            bcol[out] = c;
            for (int i = 0; i < 4; ++i) bval[4 * out + i] = v[i];
            ++out;
        }
        ++cnt;
    }
    if (!FILL) bcnt[b] = cnt;
}

static uint64_t spread3(uint64_t v) {   // 21 bits -> every third bit
    uint64_t r = 0;
    for (int i = 0; i < 21; ++i) r |= ((v >> i) & 1ULL) << (3 * i);
    return r;
}

// RWG ids in Morton order of their centres on a lattice of spacing h, padded
// with -1 to a multiple of B: consecutive rows are spatially close, so the
// near sets of a block of B rows overlap (fill ~0.75 at 4 rows).
static std::vector<int32_t> morton_rows(const aim_plan* p, int B) {
    const long long N = p->N;
    std::vector<double> cen(3 * N);
    AIM_CUDA(cudaMemcpy(cen.data(), p->rwg_c, sizeof(double) * 3 * N, cudaMemcpyDeviceToHost));
    double lo[3] = {1e300, 1e300, 1e300};
    for (long long n = 0; n < N; ++n)
        for (int a = 0; a < 3; ++a) lo[a] = std::min(lo[a], cen[3 * n + a]);
    std::vector<std::pair<uint64_t, int32_t>> key(N);
    for (long long n = 0; n < N; ++n) {
        uint64_t code = 0;
        for (int a = 0; a < 3; ++a) {
            const long long q = std::min<long long>((long long)std::floor((cen[3 * n + a] - lo[a]) / p->h), (1 << 21) - 1);
            code |= spread3((uint64_t)std::max<long long>(q, 0)) << a;
        }
        key[n] = {code, (int32_t)n};
    }
    std::stable_sort(key.begin(), key.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    const long long nblk = (N + B - 1) / B;
    std::vector<int32_t> rows(B * nblk, -1);
    for (long long n = 0; n < N; ++n) rows[n] = key[n].second;
    return rows;
}

// ------------------------- near field, 8*MT-row blocks for FP64 MMA
// Block = 8*MT Morton-consecutive rows (MT m-tiles of mma.m8n8k4); its
// columns = the sorted union of the rows' columns, cut into chunks of 4 (the
// k extent).  Chunk c stores col[4c..4c+3] (-1 = padding) and MT 32-bit masks:
// bit 4*i + k of word q says row 8q + i has column k.  The values present are
// packed in (word, bit) order, so exactly the nnzN near values are stored (no
// fill).  One thread per block.
template <bool FILL, int MT>
__global__ void near_mma_build_kernel(const int32_t* __restrict__ rows, long long nblk,
                                      const int64_t* __restrict__ rowp, const int32_t* __restrict__ col,
                                      const double2* __restrict__ val, const int64_t* __restrict__ cptr,
                                      const int64_t* __restrict__ vptr, int64_t* __restrict__ ccnt,
                                      uint32_t* __restrict__ cmask, int32_t* __restrict__ ccol,
                                      double2* __restrict__ cval) {
    constexpr int RB = 8 * MT;
    const long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nblk) return;
    long long pos[RB], end[RB];
    for (int i = 0; i < RB; ++i) {
        const int r = rows[RB * b + i];
        pos[i] = r >= 0 ? rowp[r] : 0;
        end[i] = r >= 0 ? rowp[r + 1] : 0;
    }
    long long ch = FILL ? cptr[b] : 0, vo = FILL ? vptr[b] : 0;
    long long nun = 0;
    uint32_t mask[MT];
    for (int q = 0; q < MT; ++q) mask[q] = 0;
    int k = 0;
    long long src[32 * MT];   // value index of (word q, bit 4i+k) (FILL)
    for (;;) {
        int c = INT_MAX;
        for (int i = 0; i < RB; ++i)
            if (pos[i] < end[i]) c = min(c, col[pos[i]]);
        if (c != INT_MAX) {
            for (int i = 0; i < RB; ++i)
                if (pos[i] < end[i] && col[pos[i]] == c) {
                    const int q = i / 8, bit = 4 * (i % 8) + k;
                    mask[q] |= 1u << bit;
                    src[32 * q + bit] = pos[i];
                    ++pos[i];
                }
            if (FILL) ccol[4 * ch + k] = c;
            ++k;
            ++nun;
        }
        if (k == 4 || (c == INT_MAX && k > 0)) {
            if (FILL) {
                for (int kk = k; kk < 4; ++kk) ccol[4 * ch + kk] = -1;
                for (int q = 0; q < MT; ++q) {
                    cmask[MT * ch + q] = mask[q];
                    for (int bit = 0; bit < 32; ++bit)
                        if (mask[q] >> bit & 1u) cval[vo++] = val[src[32 * q + bit]];
                }
            }
            ++ch;
            for (int q = 0; q < MT; ++q) mask[q] = 0;
            k = 0;
        }
        if (c == INT_MAX) break;
    }
    if (!FILL) ccnt[b] = (nun + 3) / 4;
}

void build_near_mma(aim_plan* p, cudaStream_t s) {
    if (p->nm_count) return;
    const long long N = p->N;
    const char* e = getenv("AIM_NEAR_RB");
    const int MT = (e && atoi(e) == 8) ? 1 : 2;   // 16-row blocks unless overridden (A/B timing)
    const int RB = 8 * MT;
    const std::vector<int32_t> rows = morton_rows(p, RB);
    const long long nblk = (long long)rows.size() / RB;
    p->nm_rows = p->alloc<int32_t>(RB * nblk);
    h2d(p->nm_rows, rows.data(), sizeof(int32_t) * RB * nblk, s);
    int64_t* d_cnt = nullptr;
    AIM_CUDA(cudaMalloc(&d_cnt, sizeof(int64_t) * nblk));
    if (MT == 1)
        near_mma_build_kernel<false, 1><<<nblk_of(nblk), 128, 0, s>>>(p->nm_rows, nblk, p->nrow, p->ncol, p->nval,
                                                                      nullptr, nullptr, d_cnt, nullptr, nullptr, nullptr);
    else
        near_mma_build_kernel<false, 2><<<nblk_of(nblk), 128, 0, s>>>(p->nm_rows, nblk, p->nrow, p->ncol, p->nval,
                                                                      nullptr, nullptr, d_cnt, nullptr, nullptr, nullptr);
    note_launch("near_mma_count");
    std::vector<int64_t> cnt(nblk), cptr(nblk + 1, 0), vptr(nblk + 1, 0), rowp(N + 1);
    AIM_CUDA(cudaMemcpyAsync(cnt.data(), d_cnt, sizeof(int64_t) * nblk, cudaMemcpyDeviceToHost, s));
    AIM_CUDA(cudaMemcpyAsync(rowp.data(), p->nrow, sizeof(int64_t) * (N + 1), cudaMemcpyDeviceToHost, s));
    AIM_CUDA(cudaStreamSynchronize(s));
    for (long long b = 0; b < nblk; ++b) {
        cptr[b + 1] = cptr[b] + cnt[b];
        long long nz = 0;
        for (int i = 0; i < RB; ++i) {
            const int r = rows[RB * b + i];
            if (r >= 0) nz += rowp[r + 1] - rowp[r];
        }
        vptr[b + 1] = vptr[b] + nz;
    }
    p->nm_chunks = cptr[nblk];
    p->nm_mt = MT;
    p->nm_cptr = p->alloc<int64_t>(nblk + 1);
    p->nm_vptr = p->alloc<int64_t>(nblk + 1);
    p->nm_mask = p->alloc<uint32_t>(MT * p->nm_chunks);
    p->nm_col = p->alloc<int32_t>(4 * p->nm_chunks);
    p->nm_val = p->alloc<double2>(p->nnzN);
    AIM_CUDA(cudaMemcpyAsync(p->nm_cptr, cptr.data(), sizeof(int64_t) * (nblk + 1), cudaMemcpyHostToDevice, s));
    AIM_CUDA(cudaMemcpyAsync(p->nm_vptr, vptr.data(), sizeof(int64_t) * (nblk + 1), cudaMemcpyHostToDevice, s));
    if (MT == 1)
        near_mma_build_kernel<true, 1><<<nblk_of(nblk), 128, 0, s>>>(p->nm_rows, nblk, p->nrow, p->ncol, p->nval,
                                                                     p->nm_cptr, p->nm_vptr, nullptr, p->nm_mask,
                                                                     p->nm_col, p->nm_val);
    else
        near_mma_build_kernel<true, 2><<<nblk_of(nblk), 128, 0, s>>>(p->nm_rows, nblk, p->nrow, p->ncol, p->nval,
                                                                     p->nm_cptr, p->nm_vptr, nullptr, p->nm_mask,
                                                                     p->nm_col, p->nm_val);
    note_launch("near_mma_fill");
    AIM_CUDA(cudaStreamSynchronize(s));
    cudaFree(d_cnt);
    p->nm_count = nblk;
}

// --------------------------------- interpolation, 8*MT-row blocks for FP64 MMA
// H5 as a block-sparse product y = jk eta0 W Phi: rows = 8*MT Morton-consecutive
// RWGs, columns = the sorted union of their stencil nodes; one chunk per node
// whose 4 k-columns are the components (x, y, z, phi).  Chunk c stores the
// node index and MT masks (bit 4i + comp: row 8q + i touches the node); the
// present weights are packed in mask order, the phi weight pre-scaled by
// -1/k^2, so y = jk eta0 sum_k A B.  Built on the host once (first
// multi-RHS interpolation).
void build_interp_mma(aim_plan* p, cudaStream_t s) {
    if (p->im_count) return;
    const long long N = p->N;
    const int M1 = p->M + 1, S = p->S, Ny = p->dims[1], Nz = p->dims[2];
    const char* e = getenv("AIM_INTERP_RB");
    const int MT = (e && atoi(e) == 8) ? 1 : 2;
    const int RB = 8 * MT;
    const std::vector<int32_t> rows = morton_rows(p, RB);
    const long long nblk = (long long)rows.size() / RB;
    std::vector<int32_t> node0(N);
    std::vector<double> W((size_t)N * S * 4);
    AIM_CUDA(cudaStreamSynchronize(s));
    AIM_CUDA(cudaMemcpy(node0.data(), p->node0, sizeof(int32_t) * N, cudaMemcpyDeviceToHost));
    AIM_CUDA(cudaMemcpy(W.data(), p->W, sizeof(double) * W.size(), cudaMemcpyDeviceToHost));
    const double ik2 = 1.0 / (p->k * p->k);
    std::vector<int64_t> cptr(nblk + 1, 0), vptr(nblk + 1, 0);
    std::vector<int32_t> cnode;
    std::vector<uint32_t> cmask;
    std::vector<double> cval;
    cnode.reserve(N * 8);
    cval.reserve((size_t)N * S * 4);
    std::vector<int32_t> nodes;
    auto coords = [&](long long g, int& x, int& y, int& z) {
        z = (int)(g % Nz);
        y = (int)((g / Nz) % Ny);
        x = (int)(g / ((long long)Ny * Nz));
    };
    for (long long b = 0; b < nblk; ++b) {
        nodes.clear();
        for (int i = 0; i < RB; ++i) {
            const int r = rows[RB * b + i];
            if (r < 0) continue;
            int bx, by, bz;
            coords(node0[r], bx, by, bz);
            for (int u = 0; u < S; ++u) {
                const int ux = u / (M1 * M1), uy = (u / M1) % M1, uz = u % M1;
                nodes.push_back((int32_t)(((long long)(bx + ux) * Ny + (by + uy)) * Nz + (bz + uz)));
            }
        }
        std::sort(nodes.begin(), nodes.end());
        nodes.erase(std::unique(nodes.begin(), nodes.end()), nodes.end());
        for (int32_t g : nodes) {
            int gx, gy, gz;
            coords(g, gx, gy, gz);
            cnode.push_back(g);
            for (int q = 0; q < MT; ++q) {
                uint32_t m = 0;
                for (int i = 0; i < 8; ++i) {
                    const int r = rows[RB * b + 8 * q + i];
                    if (r < 0) continue;
                    int bx, by, bz;
                    coords(node0[r], bx, by, bz);
                    const int dx = gx - bx, dy = gy - by, dz = gz - bz;
                    if (dx < 0 || dx > p->M || dy < 0 || dy > p->M || dz < 0 || dz > p->M) continue;
                    const int u = (dx * M1 + dy) * M1 + dz;
                    m |= 0xFu << (4 * i);
                    const double* w = &W[((size_t)r * S + u) * 4];
                    cval.push_back(w[0]);
                    cval.push_back(w[1]);
                    cval.push_back(w[2]);
                    cval.push_back(-w[3] * ik2);
                }
                cmask.push_back(m);
            }
        }
        cptr[b + 1] = (int64_t)cnode.size();
        vptr[b + 1] = (int64_t)cval.size();
    }
    if ((long long)cval.size() >= (1LL << 31)) throw Error(AIM_E_GRID, "interp_mma: packed weights exceed 2^31");
    p->im_mt = MT;
    p->im_chunks = (int64_t)cnode.size();
    p->im_rows = p->alloc<int32_t>(rows.size());
    p->im_cptr = p->alloc<int64_t>(nblk + 1);
    p->im_vptr = p->alloc<int64_t>(nblk + 1);
    p->im_node = p->alloc<int32_t>(cnode.size());
    p->im_mask = p->alloc<uint32_t>(cmask.size());
    p->im_val = p->alloc<double>(cval.size());
    h2d(p->im_rows, rows.data(), sizeof(int32_t) * rows.size(), s);
    h2d(p->im_cptr, cptr.data(), sizeof(int64_t) * (nblk + 1), s);
    h2d(p->im_vptr, vptr.data(), sizeof(int64_t) * (nblk + 1), s);
    h2d(p->im_node, cnode.data(), sizeof(int32_t) * cnode.size(), s);
    h2d(p->im_mask, cmask.data(), sizeof(uint32_t) * cmask.size(), s);
    h2d(p->im_val, cval.data(), sizeof(double) * cval.size(), s);
    p->im_count = nblk;
}

void build_near_blocks(aim_plan* p, cudaStream_t s) {
    if (p->nb_count) return;
    const std::vector<int32_t> rows = morton_rows(p, 4);
    const long long nblk = (long long)rows.size() / 4;
    p->nb_rows = p->alloc<int32_t>(4 * nblk);
    h2d(p->nb_rows, rows.data(), sizeof(int32_t) * 4 * nblk, s);
    int64_t* d_cnt = nullptr;
    AIM_CUDA(cudaMalloc(&d_cnt, sizeof(int64_t) * nblk));
    near_block_kernel<false><<<nblk_of(nblk), 128, 0, s>>>(p->nb_rows, nblk, p->nrow, p->ncol, p->nval, nullptr, d_cnt,
                                                           nullptr, nullptr);
    note_launch("near_block_count");
    std::vector<int64_t> cnt(nblk), ptr(nblk + 1, 0);
    AIM_CUDA(cudaMemcpyAsync(cnt.data(), d_cnt, sizeof(int64_t) * nblk, cudaMemcpyDeviceToHost, s));
    AIM_CUDA(cudaStreamSynchronize(s));
    for (long long b = 0; b < nblk; ++b) ptr[b + 1] = ptr[b] + cnt[b];
    p->nbc = ptr[nblk];
    p->nb_ptr = p->alloc<int64_t>(nblk + 1);
    p->nb_col = p->alloc<int32_t>(p->nbc);
    p->nb_val = p->alloc<double2>(4 * p->nbc);
    AIM_CUDA(cudaMemcpyAsync(p->nb_ptr, ptr.data(), sizeof(int64_t) * (nblk + 1), cudaMemcpyHostToDevice, s));
    near_block_kernel<true><<<nblk_of(nblk), 128, 0, s>>>(p->nb_rows, nblk, p->nrow, p->ncol, p->nval, p->nb_ptr,
                                                          nullptr, p->nb_col, p->nb_val);
    note_launch("near_block_fill");
    AIM_CUDA(cudaStreamSynchronize(s));
    cudaFree(d_cnt);
    p->nb_count = nblk;
    if (p->prec == AIM_C64) make_c64_blocks(p, s);
}

// ------------------------------------------------------- S4 exact entries
struct NearArgs {
    const double* qp;      // [nt][7][3]
    const double* qw;      // [nt][7]
    const double* cor;     // [nt][3][3]
    const int32_t* tv;     // [nt][3]
    const int32_t* rt;     // [N][2]
    const double* ra;      // [N][2]
    const double* rp;      // [N][2][3]
    const int32_t* base;   // [N][3]
    const double* W;       // [N][S][4]
    const int64_t* rowp;
    const int32_t* col;
    double2* val;
    const double2* htab;   // [(D+1)^3] G(h |d|), G(0)=0
    int D;
    long long N;
    double k, h, keta;     // keta = k eta0
};

struct Mom {
    double2 I00, I11;
    double2 I10[3], I01[3];
};

__device__ __forceinline__ double2 green_full(double R, double k) {
    double s, c;
    sincos(k * R, &s, &c);
    const double f = 1.0 / (4.0 * kPi * R);
    return make_double2(c * f, -s * f);
}

// G_s(R) = (exp(-jkR) - 1)/(4 pi R) = (-2 sin^2(kR/2) - j sin kR)/(4 pi R); G_s(0) = -jk/(4 pi)
__device__ __forceinline__ double2 green_smooth(double R, double k) {
    if (R == 0.0) return make_double2(0.0, -k / (4.0 * kPi));
    const double sh = sin(0.5 * k * R);
    const double f = 1.0 / (4.0 * kPi * R);
    return make_double2(-2.0 * sh * sh * f, -sin(k * R) * f);
}

// Static potentials over the flat triangle cor[0..2] seen from r:
//   J0 = int 1/R dS',  Jr = int r'/R dS'  (D8 closed forms)
__device__ void static_pot(const double* r, const double* cor, double& J0, double Jr[3]) {
    const double* v1 = cor;
    const double* v2 = cor + 3;
    const double* v3 = cor + 6;
    double e1[3] = {v2[0] - v1[0], v2[1] - v1[1], v2[2] - v1[2]};
    double e2[3] = {v3[0] - v1[0], v3[1] - v1[1], v3[2] - v1[2]};
    double nv[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2], e1[0] * e2[1] - e1[1] * e2[0]};
    const double nn = sqrt(nv[0] * nv[0] + nv[1] * nv[1] + nv[2] * nv[2]);
    nv[0] /= nn; nv[1] /= nn; nv[2] /= nn;
    const double d = nv[0] * (r[0] - v1[0]) + nv[1] * (r[1] - v1[1]) + nv[2] * (r[2] - v1[2]);
    const double rho[3] = {r[0] - d * nv[0], r[1] - d * nv[1], r[2] - d * nv[2]};
    const double ad = fabs(d);
    double I0 = 0.0, I1[3] = {0.0, 0.0, 0.0};
    const double* A[3] = {v1, v2, v3};
    const double* B[3] = {v2, v3, v1};
    for (int e = 0; e < 3; ++e) {
        const double* a = A[e];
        const double* b = B[e];
        double lv[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
        const double le = sqrt(lv[0] * lv[0] + lv[1] * lv[1] + lv[2] * lv[2]);
        lv[0] /= le; lv[1] /= le; lv[2] /= le;
        const double u[3] = {lv[1] * nv[2] - lv[2] * nv[1], lv[2] * nv[0] - lv[0] * nv[2], lv[0] * nv[1] - lv[1] * nv[0]};
        const double lp = (b[0] - rho[0]) * lv[0] + (b[1] - rho[1]) * lv[1] + (b[2] - rho[2]) * lv[2];
        const double lm = (a[0] - rho[0]) * lv[0] + (a[1] - rho[1]) * lv[1] + (a[2] - rho[2]) * lv[2];
        const double P0 = (a[0] - rho[0]) * u[0] + (a[1] - rho[1]) * u[1] + (a[2] - rho[2]) * u[2];
        const double R0sq = P0 * P0 + d * d;
        const double Rp = sqrt((r[0] - b[0]) * (r[0] - b[0]) + (r[1] - b[1]) * (r[1] - b[1]) + (r[2] - b[2]) * (r[2] - b[2]));
        const double Rm = sqrt((r[0] - a[0]) * (r[0] - a[0]) + (r[1] - a[1]) * (r[1] - a[1]) + (r[2] - a[2]) * (r[2] - a[2]));
        double f = 0.0;
        if (R0sq > (1e-12 * le) * (1e-12 * le)) {
            const double np_ = lp >= 0 ? Rp + lp : R0sq / (Rp - lp);
            const double nm_ = lm >= 0 ? Rm + lm : R0sq / (Rm - lm);
            f = log(np_ / nm_);
        }
        I0 += P0 * f - ad * (atan2(P0 * lp, R0sq + ad * Rp) - atan2(P0 * lm, R0sq + ad * Rm));
        const double c = 0.5 * (R0sq * f + lp * Rp - lm * Rm);
        I1[0] += c * u[0];
        I1[1] += c * u[1];
        I1[2] += c * u[2];
    }
    J0 = I0;
    Jr[0] = I1[0] + rho[0] * I0;
    Jr[1] = I1[1] + rho[1] * I0;
    Jr[2] = I1[2] + rho[2] * I0;
}

// Moments of the triangle pair (t test/outer, tp source/inner)
__device__ void pair_moments(const NearArgs& a, int t, int tp, bool sing, Mom& m) {
    m.I00 = m.I11 = make_double2(0, 0);
    for (int c = 0; c < 3; ++c) m.I10[c] = m.I01[c] = make_double2(0, 0);
    for (int q = 0; q < 7; ++q) {
        const double* rq = a.qp + (7 * t + q) * 3;
        const double wq = a.qw[7 * t + q];
        double2 in0 = make_double2(0, 0);
        double2 in1[3] = {make_double2(0, 0), make_double2(0, 0), make_double2(0, 0)};
        for (int pp = 0; pp < 7; ++pp) {
            const double* rpt = a.qp + (7 * tp + pp) * 3;
            const double wp = a.qw[7 * tp + pp];
            const double dx = rq[0] - rpt[0], dy = rq[1] - rpt[1], dz = rq[2] - rpt[2];
            const double R = sqrt(dx * dx + dy * dy + dz * dz);
            const double2 g = sing ? green_smooth(R, a.k) : green_full(R, a.k);
            const double2 gw = make_double2(g.x * wp, g.y * wp);
            in0.x += gw.x; in0.y += gw.y;
            for (int c = 0; c < 3; ++c) { in1[c].x += gw.x * rpt[c]; in1[c].y += gw.y * rpt[c]; }
        }
        if (sing) {
            double J0, Jr[3];
            static_pot(rq, a.cor + 9 * tp, J0, Jr);
            const double s = 1.0 / (4.0 * kPi);
            in0.x += J0 * s;
            for (int c = 0; c < 3; ++c) in1[c].x += Jr[c] * s;
        }
        m.I00.x += wq * in0.x; m.I00.y += wq * in0.y;
        for (int c = 0; c < 3; ++c) {
            m.I10[c].x += wq * in0.x * rq[c]; m.I10[c].y += wq * in0.y * rq[c];
            m.I01[c].x += wq * in1[c].x;      m.I01[c].y += wq * in1[c].y;
            m.I11.x += wq * rq[c] * in1[c].x; m.I11.y += wq * rq[c] * in1[c].y;
        }
    }
}

// alpha beta [I11 - pn.I10 - pm.I01 + (pm.pn) I00] - k^-2 (2 alpha)(2 beta) I00   (without j k eta0)
__device__ __forceinline__ double2 combine(const Mom& m, double al, double be, const double* pm, const double* pn,
                                           double k) {
    double2 lam = m.I11;
    const double pp = pm[0] * pn[0] + pm[1] * pn[1] + pm[2] * pn[2];
    lam.x += pp * m.I00.x; lam.y += pp * m.I00.y;
    for (int c = 0; c < 3; ++c) {
        lam.x -= pn[c] * m.I10[c].x + pm[c] * m.I01[c].x;
        lam.y -= pn[c] * m.I10[c].y + pm[c] * m.I01[c].y;
    }
    const double ab = al * be;
    const double ch = 4.0 * ab / (k * k);
    return make_double2(ab * lam.x - ch * m.I00.x, ab * lam.y - ch * m.I00.y);
}

__device__ __forceinline__ bool share_vertex(const int32_t* tv, int t, int tp) {
    bool s = false;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) s |= (tv[3 * t + i] == tv[3 * tp + j]);
    return s;
}

// Z_ex_sym[m,n] / (j k eta0): regular triangle pairs are symmetric under
// swapping test and source (same 7x7 products), singular ones are averaged.
__device__ double2 exact_sym(const NearArgs& a, long long m, long long n) {
    double2 z = make_double2(0, 0);
    for (int sm = 0; sm < 2; ++sm)
        for (int sn = 0; sn < 2; ++sn) {
            const int t = a.rt[2 * m + sm], tp = a.rt[2 * n + sn];
            const double al = a.ra[2 * m + sm], be = a.ra[2 * n + sn];
            const double* pm = a.rp + 6 * m + 3 * sm;
            const double* pn = a.rp + 6 * n + 3 * sn;
            Mom mo;
            const bool sing = share_vertex(a.tv, t, tp);
            pair_moments(a, t, tp, sing, mo);
            double2 c = combine(mo, al, be, pm, pn, a.k);
            if (sing) {
                Mom mt;
                pair_moments(a, tp, t, true, mt);  // test on n's triangle, source on m's
                const double2 c2 = combine(mt, be, al, pn, pm, a.k);
                c = make_double2(0.5 * (c.x + c2.x), 0.5 * (c.y + c2.y));
            }
            z.x += c.x; z.y += c.y;
        }
    return z;
}

// warp per row m, lanes over the row's near entries
template <int M>
__global__ void __launch_bounds__(256) near_values_kernel(NearArgs a) {
    constexpr int M1 = M + 1, S = M1 * M1 * M1;
    extern __shared__ double2 sh[];
    const int D1 = a.D + 1;
    const int ntab = D1 * D1 * D1;
    double2* htab = sh;
    double* wm_all = reinterpret_cast<double*>(sh + ntab);
    for (int i = threadIdx.x; i < ntab; i += blockDim.x) htab[i] = a.htab[i];
    __syncthreads();
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    const long long m = (long long)blockIdx.x * (blockDim.x / 32) + warp;
    if (m >= a.N) return;
    double* wm = wm_all + warp * S * 4;
    for (int i = lane; i < S * 4; i += 32) wm[i] = a.W[m * S * 4 + i];
    __syncwarp();
    const int bmx = a.base[3 * m], bmy = a.base[3 * m + 1], bmz = a.base[3 * m + 2];
    for (long long e = a.rowp[m] + lane; e < a.rowp[m + 1]; e += 32) {
        const long long n = a.col[e];
        // grid part w_m^T H w_n (xyz) and (phi)
        const int dx0 = bmx - a.base[3 * n], dy0 = bmy - a.base[3 * n + 1], dz0 = bmz - a.base[3 * n + 2];
        double2 accA = make_double2(0, 0), accP = make_double2(0, 0);
        const double* wn = a.W + n * S * 4;
        for (int v = 0; v < S; ++v) {
            const double2 w01 = __ldg(reinterpret_cast<const double2*>(wn + 4 * v));
            const double2 w23 = __ldg(reinterpret_cast<const double2*>(wn + 4 * v) + 1);
            const int vi = v / (M1 * M1), vj = (v / M1) % M1, vk = v % M1;
#pragma unroll 4
            for (int u = 0; u < S; ++u) {
                const int ui = u / (M1 * M1), uj = (u / M1) % M1, uk = u % M1;
                const int ix = abs(dx0 + ui - vi), iy = abs(dy0 + uj - vj), iz = abs(dz0 + uk - vk);
                double2 H;
                if (ix <= a.D && iy <= a.D && iz <= a.D) {
                    H = htab[(ix * D1 + iy) * D1 + iz];
                } else {
                    const double R = a.h * sqrt((double)(ix * ix + iy * iy + iz * iz));
                    H = green_full(R, a.k);
                }
                const double* w = wm + 4 * u;
                const double s3 = w[0] * w01.x + w[1] * w01.y + w[2] * w23.x;
                const double s1 = w[3] * w23.y;
                accA.x += H.x * s3; accA.y += H.y * s3;
                accP.x += H.x * s1; accP.y += H.y * s1;
            }
        }
        const double ik2 = 1.0 / (a.k * a.k);
        const double2 grid = make_double2(accA.x - accP.x * ik2, accA.y - accP.y * ik2);
        const double2 ex = exact_sym(a, m, n);
        const double2 d = make_double2(ex.x - grid.x, ex.y - grid.y);
        // j k eta0 * d
        a.val[e] = make_double2(-a.keta * d.y, a.keta * d.x);
    }
}

__global__ void htab_kernel(double2* tab, int D, double h, double k) {
    const int D1 = D + 1;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= D1 * D1 * D1) return;
    const int x = i / (D1 * D1), y = (i / D1) % D1, z = i % D1;
    const int q = x * x + y * y + z * z;
    tab[i] = q == 0 ? make_double2(0, 0) : green_full(h * sqrt((double)q), k);
}

void build_near_values(aim_plan* p, cudaStream_t s) {
    p->nval = p->alloc<double2>(p->nnzN + 1);
    p->ncol_padded = 1;
    const double lim = p->r * (1.0 + 1e-9);
    // table of G(h|d|) over |d_a| <= D in shared memory; offsets beyond the
    // table (huge near radii) fall back to direct evaluation in the kernel
    const int D = std::min((int)std::floor(lim / p->h) + 1 + p->M, 15);
    const int D1 = D + 1;
    double2* htab = nullptr;
    AIM_CUDA(cudaMalloc(&htab, sizeof(double2) * D1 * D1 * D1));
    htab_kernel<<<nblk(D1 * D1 * D1, 256), 256, 0, s>>>(htab, D, p->h, p->k);
    note_launch("htab");
    NearArgs a;
    a.qp = p->tri_qp; a.qw = p->tri_qw; a.cor = p->tri_cor; a.tv = p->tri_v;
    a.rt = p->rwg_t; a.ra = p->rwg_a; a.rp = p->rwg_p; a.base = p->base; a.W = p->W;
    a.rowp = p->nrow; a.col = p->ncol; a.val = p->nval; a.htab = htab; a.D = D;
    a.N = p->N; a.k = p->k; a.h = p->h; a.keta = p->k * eta0();
    const int threads = 256, warps = threads / 32;
    const size_t smem = sizeof(double2) * D1 * D1 * D1 + sizeof(double) * warps * p->S * 4;
    switch (p->M) {
#define NV_CASE(MM)                                                                                       \
    case MM:                                                                                              \
        AIM_CUDA(cudaFuncSetAttribute(near_values_kernel<MM>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                      (int)std::max<size_t>(smem, 48 * 1024)));                         \
        near_values_kernel<MM><<<nblk(p->N, warps), threads, smem, s>>>(a);                                \
        break;
        NV_CASE(1) NV_CASE(2) NV_CASE(3) NV_CASE(4) NV_CASE(5) NV_CASE(6)
#undef NV_CASE
    }
    note_launch("near_values");
    AIM_CUDA(cudaStreamSynchronize(s));
    cudaFree(htab);
}

// ------------------------------------------------------ S3 Green spectrum
// K[x][y][z] = G(h sqrt(xb^2 + yb^2 + zb^2)), xb = min(x, Px - x) (min image,
// D12) for z < Lz; zb = min(z, Pz - z) in 3-D mode, zb = z (the |dz| of the
// direct z convolution) in planar mode.
__global__ void kernel_sample(double2* K, int Px, int Py, int Lz, int Pz, int planar, double h, double k) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long tot = (long long)Px * Py * Lz;
    if (i >= tot) return;
    const int x = (int)(i / ((long long)Py * Lz)), y = (int)((i / Lz) % Py), z = (int)(i % Lz);
    const int ix = min(x, Px - x), iy = min(y, Py - y), iz = planar ? z : min(z, Pz - z);
    const double q = (double)ix * ix + (double)iy * iy + (double)iz * iz;
    K[i] = q == 0 ? make_double2(0, 0) : green_full(h * sqrt(q), k);
}

// spec[(x PyH + y) Lo + z] = F[x][y][z] * scale for x <= Px/2, y <= Py/2, z < Lo
__global__ void spectrum_octant(const double2* F, double2* spec, int Px, int Py, int Lz, int Lo, double scale) {
    const int PxH = Px / 2 + 1, PyH = Py / 2 + 1;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)PxH * PyH * Lo) return;
    const int x = (int)(i / ((long long)PyH * Lo)), y = (int)((i / Lo) % PyH), z = (int)(i % Lo);
    const double2 v = F[((long long)x * Py + y) * Lz + z];
    spec[i] = make_double2(v.x * scale, v.y * scale);
}

void build_green_spectrum(aim_plan* p, cudaStream_t s) {
    const int Px = p->pads[0], Py = p->pads[1], Pz = p->pads[2], Nz = p->dims[2];
    const int Lz = p->planar ? Nz : Pz;   // modes 1 and 2 share the 2-D spectrum G2(kx, ky, dz)
    const long long tot = (long long)Px * Py * Lz;
    double2 *A = nullptr, *B = nullptr;
    AIM_CUDA(cudaMalloc(&A, sizeof(double2) * tot));
    AIM_CUDA(cudaMalloc(&B, sizeof(double2) * tot));
    kernel_sample<<<nblk(tot, 256), 256, 0, s>>>(A, Px, Py, Lz, Pz, p->planar, p->h, p->k);
    note_launch("kernel_sample");
    FftPass f{};
    f.mode = 0;
    // x: [1][Px][Py Lz]
    f.in = A; f.out = B; f.outer = 1; f.Lin = f.Lout = Px; f.inner = (long long)Py * Lz; f.ax = p->ax[0];
    f.TO = f.TI = 0;
    launch_fft_pass(f, s);
    // y: [Px][Py][Lz]
    f.in = B; f.out = A; f.outer = Px; f.Lin = f.Lout = Py; f.inner = Lz; f.ax = p->ax[1];
    f.TO = f.TI = 0;
    launch_fft_pass(f, s);
    double2* F = A;
    double scale = 1.0 / ((double)Px * Py);
    int Lo = Nz;
    if (!p->planar) {
        // z: [Px Py][Pz][1]
        f.in = A; f.out = B; f.outer = (long long)Px * Py; f.Lin = f.Lout = Pz; f.inner = 1; f.ax = p->ax[2];
        f.TO = f.TI = 0;
        launch_fft_pass(f, s);
        F = B;
        scale /= (double)Pz;
        Lo = Pz / 2 + 1;
    }
    const long long oct = (long long)(Px / 2 + 1) * (Py / 2 + 1) * Lo;
    p->spec = p->alloc<double2>(oct);
    p->spec_len = oct;
    spectrum_octant<<<nblk(oct, 256), 256, 0, s>>>(F, p->spec, Px, Py, Lz, Lo, scale);
    note_launch("spectrum_octant");
    AIM_CUDA(cudaStreamSynchronize(s));
    cudaFree(A);
    cudaFree(B);
}

}  // namespace aim

namespace aim {

// Dense element block for the block-Jacobi preconditioner (k_precond.cu):
// out[i][j] = Z_ex_sym[rows[i], rows[j]] (j k eta0 included), all pairs of the
// element, the same exact Galerkin entries as the near field (D8, D9).
__global__ void exact_block_kernel(NearArgs a, const int32_t* __restrict__ rows, int n, double2* __restrict__ out) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)n * n) return;
    const int i = (int)(e / n), j = (int)(e - (e / n) * n);
    const double2 z = exact_sym(a, rows[i], rows[j]);
    out[e] = make_double2(-a.keta * z.y, a.keta * z.x);
}

void fill_exact_block(aim_plan* p, const int32_t* d_rows, int n, double2* d_out, cudaStream_t s) {
    NearArgs a{};
    a.qp = p->tri_qp; a.qw = p->tri_qw; a.cor = p->tri_cor; a.tv = p->tri_v;
    a.rt = p->rwg_t; a.ra = p->rwg_a; a.rp = p->rwg_p;
    a.N = p->N; a.k = p->k; a.h = p->h; a.keta = p->k * eta0();
    const long long tot = (long long)n * n;
    exact_block_kernel<<<(unsigned)((tot + 127) / 128), 128, 0, s>>>(a, d_rows, n, d_out);
    note_launch("exact_block");
}

}  // namespace aim
