// Restarted GMRES on the device (PAPER.md:510-511
// "we solve the linear system ... iteratively using the generalized minimal
// residual (GMRES) algorithm"; reading D15).
//
// Krylov basis V [restart+1][n] and all vector work stay in HBM; the host
// keeps only the (restart+1) x restart Hessenberg matrix and the Givens
// rotations.  Arnoldi is classical Gram-Schmidt applied twice (CGS2) in three
// passes over the basis per iteration (DESIGN.md §5 "GMRES"):
//   pass 1  h1 = V^H w                                   (mdot_kernel)
//   pass 2  w -= V h1, then h2 = V^H w, V read once      (axpy_dot_smem_kernel)
//   pass 3  w -= V h2 and ||w||^2                        (axpy_norm_kernel)
// then v_{j+1} = w / ||w||.  Every coefficient is produced and consumed on
// the device (fixed-order block partials -> deterministic); the host reads
// h1, h2, ||w|| once per iteration (one synchronisation) for the Givens
// rotations and the convergence test.  Distributed use: `allreduce` sums the
// small coefficient vectors over the ranks between the partial and the use,
// with the Krylov vectors partitioned by owning rank (k_slab.cu).
// Right preconditioning (optional): A M^-1 u = b, x = M^-1 u.
#include <math.h>

#include <algorithm>
#include <complex>
#include <functional>
#include <vector>

#include "aim_internal.cuh"

namespace aim {

using cplx = std::complex<double>;

static constexpr int kGmBlocks = 296;   // 2 x 148 SMs
static constexpr int kAdBlocks = 296;   // axpy_dot_smem_kernel: 2 x 148 SMs (3 measured slower)
static constexpr int kAnBlocks = 2368;  // axpy_norm_kernel: up to 16 x 148 blocks of 256 threads
static constexpr int kPartBlocks = kAnBlocks;   // rows of the block-partials buffer
static constexpr int kGmThreads = 512;  // 16 warps
static constexpr int kGmWarps = kGmThreads / 32;
static constexpr int kGmChunk = 64;     // basis vectors per pass
static constexpr int kGmQ = kGmChunk / kGmWarps;   // basis vectors per warp (4)
static constexpr int kMaxBasis = 1024;

__device__ __forceinline__ void cfma_conj(double2& acc, double2 v, double2 x) {   // acc += conj(v) x
    acc.x = fma(v.x, x.x, fma(v.y, x.y, acc.x));
    acc.y = fma(v.x, x.y, fma(-v.y, x.x, acc.y));
}
__device__ __forceinline__ void cfma(double2& acc, double2 c, double2 v) {        // acc += c v
    acc.x = fma(c.x, v.x, fma(-c.y, v.y, acc.x));
    acc.y = fma(c.x, v.y, fma(c.y, v.x, acc.y));
}
__device__ __forceinline__ double2 warp_sum(double2 s) {
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        s.x += __shfl_xor_sync(0xffffffffu, s.x, off);
        s.y += __shfl_xor_sync(0xffffffffu, s.y, off);
    }
    return s;
}

// partial[b][i] = sum_{e in block b's range} conj(V_i[e]) w[e], i < nv (nv <= 64).
// 16 warps; warp g owns basis vectors i = g + 16 q (q < 4); each lane takes
// U elements per step (e = base + lane + 32 u) so U x 4 loads are in flight;
// w[e] is read from HBM once per block (the other warps hit L1).
template <int U>
__global__ void __launch_bounds__(kGmThreads) mdot_kernel(const double2* __restrict__ V, long long ld, long long n,
                                                          int nv, const double2* __restrict__ w,
                                                          double2* __restrict__ partial) {
    const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
    const long long chunk = ((n + gridDim.x - 1) / gridDim.x + 32 * U - 1) / (32 * U) * (32 * U);
    const long long a = blockIdx.x * chunk, b = min(n, a + chunk);
    double2 acc[kGmQ];
#pragma unroll
    for (int q = 0; q < kGmQ; ++q) acc[q] = make_double2(0, 0);
    if (g < nv) {
        for (long long e0 = a + lane; e0 < b; e0 += 32 * U) {
            double2 x[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const long long e = e0 + 32 * u;
                x[u] = e < b ? __ldg(&w[e]) : make_double2(0, 0);
            }
#pragma unroll
            for (int q = 0; q < kGmQ; ++q) {
                const int i = g + kGmWarps * q;
                if (i < nv) {
                    double2 v[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const long long e = e0 + 32 * u;
                        v[u] = e < b ? __ldcs(&V[i * ld + e]) : make_double2(0, 0);
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) cfma_conj(acc[q], v[u], x[u]);
                }
            }
        }
    }
#pragma unroll
    for (int q = 0; q < kGmQ; ++q) {
        const int i = g + kGmWarps * q;
        const double2 s = warp_sum(acc[q]);
        if (lane == 0 && i < nv) partial[(long long)blockIdx.x * kGmChunk + i] = s;
    }
}

// w -= sum_i c[i] V_i (c on the device), then partial dots of the updated w
// with every V_i, V read from HBM once: the V tile is staged in shared memory
// by cp.async, double buffered: tile t+1 (nv x 64 elements, and w) lands while tile t is used.
// Per tile: thread (group q = tid / 64, element t = tid % 64) forms
// sum_{i = q mod 4} c_i V_i[e]; 64 threads rebuild w' = w - sum of the 4
// group sums; then warp g accumulates conj(V_i[e]) w'[e] for i = g mod 8
// (lanes over the 64 elements).
constexpr int kAdT = 64, kAdThreads = 256;
__device__ __forceinline__ void cp16(void* sdst, const void* gsrc, bool valid) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gsrc), "r"(valid ? 16 : 0)
                 : "memory");
}
__global__ void __launch_bounds__(kAdThreads, 2) axpy_dot_smem_kernel(const double2* __restrict__ V, long long ld,
                                                                      long long n, int nv,
                                                                      const double2* __restrict__ c,
                                                                      double2* __restrict__ w,
                                                                      double2* __restrict__ partial) {
    extern __shared__ __align__(16) double2 sm[];
    double2* buf[2] = {sm, sm + (nv + 1) * kAdT};    // [nv + 1][kAdT]: V rows then w
    __shared__ double2 red[4][kAdT];
    __shared__ double2 xs[kAdT];
    __shared__ double2 cs[kGmChunk];
    const int tid = threadIdx.x, lane = tid & 31, g = tid >> 5;
    if (tid < nv) cs[tid] = c[tid];
    const long long chunk = ((n + gridDim.x - 1) / gridDim.x + kAdT - 1) / kAdT * kAdT;
    const long long a = blockIdx.x * chunk, b = min(n, a + chunk);
    const int ntiles = b > a ? (int)((b - a + kAdT - 1) / kAdT) : 0;
    auto issue = [&](int t, double2* dst) {
        const long long e0 = a + (long long)t * kAdT;
        for (int q = tid; q < (nv + 1) * kAdT; q += kAdThreads) {
            const int i = q / kAdT, el = q - (q / kAdT) * kAdT;
            const long long e = e0 + el;
            const bool v = e < b;
            const double2* src = i < nv ? V + i * ld + (v ? e : 0) : w + (v ? e : 0);
            cp16(&dst[q], src, v);
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    double2 acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = make_double2(0, 0);
    if (ntiles) issue(0, buf[0]);
    for (int t = 0; t < ntiles; ++t) {
        double2* cur = buf[t & 1];
        if (t + 1 < ntiles) {
            issue(t + 1, buf[(t + 1) & 1]);
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        __syncthreads();
        {
            const int q = tid / kAdT, el = tid - (tid / kAdT) * kAdT;
            double2 s = make_double2(0, 0);
            for (int i = q; i < nv; i += 4) cfma(s, cs[i], cur[i * kAdT + el]);
            red[q][el] = s;
        }
        __syncthreads();
        if (tid < kAdT) {
            double2 x = cur[nv * kAdT + tid];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                x.x -= red[q][tid].x;
                x.y -= red[q][tid].y;
            }
            xs[tid] = x;
            const long long e = a + (long long)t * kAdT + tid;
            if (e < b) w[e] = x;
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int i = g + 8 * q;
            if (i < nv) {
                cfma_conj(acc[q], cur[i * kAdT + lane], xs[lane]);
                cfma_conj(acc[q], cur[i * kAdT + lane + 32], xs[lane + 32]);
            }
        }
        __syncthreads();   // buffer `cur` is refilled by the issue of tile t + 2
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int i = g + 8 * q;
        const double2 s = warp_sum(acc[q]);
        if (lane == 0 && i < nv) partial[(long long)blockIdx.x * kGmChunk + i] = s;
    }
}

// w -= sum_i c[i] V_i, and partial[b] = sum |w|^2 over block b's elements
// (thread per element -- 256-thread blocks, up to 16 per SM, grid-stride over
// the elements -- coefficients staged in shared memory).
constexpr int kAnThreads = 256;
__global__ void __launch_bounds__(kAnThreads) axpy_norm_kernel(const double2* __restrict__ V, long long ld,
                                                               long long n, int nv, const double2* __restrict__ c,
                                                               double2* __restrict__ w,
                                                               double2* __restrict__ partial, int want_norm) {
    __shared__ double2 cs[kGmChunk];
    __shared__ double red[kAnThreads / 32];
    if (threadIdx.x < nv) cs[threadIdx.x] = c[threadIdx.x];
    __syncthreads();
    double nrm = 0.0;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
        double2 x = w[e];
#pragma unroll 8
        for (int i = 0; i < nv; ++i) {
            const double2 ci = cs[i];
            const double2 v = __ldcs(&V[i * ld + e]);
            x.x -= ci.x * v.x - ci.y * v.y;
            x.y -= ci.x * v.y + ci.y * v.x;
        }
        w[e] = x;
        nrm = fma(x.x, x.x, fma(x.y, x.y, nrm));
    }
    if (!want_norm) return;
#pragma unroll
    for (int off = 16; off; off >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, off);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = nrm;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0;
        for (int q = 0; q < kAnThreads / 32; ++q) t += red[q];
        partial[(long long)blockIdx.x * kGmChunk] = make_double2(t, 0.0);
    }
}

// out[i] (+)= sum_b partial[b][i], blocks in order (deterministic).
// Warp per i: lane l sums blocks l, l + 32, ..., then a fixed shuffle tree.
__global__ void gm_reduce_kernel(const double2* __restrict__ partial, int nb, int nv, double2* __restrict__ out,
                                 int accumulate) {
    const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (i >= nv) return;
    double2 t = make_double2(0, 0);
    for (int b = lane; b < nb; b += 32) {
        const double2 v = partial[(long long)b * kGmChunk + i];
        t.x += v.x;
        t.y += v.y;
    }
    t = warp_sum(t);
    if (lane) return;
    if (accumulate) {
        out[i].x += t.x;
        out[i].y += t.y;
    } else {
        out[i] = t;
    }
}

// dst = src / sqrt(nrm2->x)   (nrm2 on the device)
// dst = src / sqrt(nrm2), and the same into dst2 when given (the fixed
// product input of the unpreconditioned solve)
__global__ void gm_scale_kernel(const double2* __restrict__ src, long long n, const double2* __restrict__ nrm2,
                                double2* __restrict__ dst, double2* __restrict__ dst2) {
    const double s = 1.0 / sqrt(nrm2->x);
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < n) {
        const double2 v = make_double2(src[e].x * s, src[e].y * s);
        dst[e] = v;
        if (dst2) dst2[e] = v;
    }
}

// out (+)= sum_i y[i] V_i
__global__ void gm_combine_kernel(const double2* __restrict__ V, long long ld, long long n, int nv,
                                  const double2* __restrict__ y, double2* __restrict__ out, int accumulate) {
    __shared__ double2 ys[kGmChunk];
    if (threadIdx.x < nv) ys[threadIdx.x] = y[threadIdx.x];
    __syncthreads();
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    double2 acc = accumulate ? out[e] : make_double2(0, 0);
    for (int i = 0; i < nv; ++i) cfma(acc, ys[i], V[i * ld + e]);
    out[e] = acc;
}

// r = b - Ax
__global__ void residual_kernel(const double2* __restrict__ b, const double2* __restrict__ Ax, long long n,
                                double2* __restrict__ r) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < n) r[e] = make_double2(b[e].x - Ax[e].x, b[e].y - Ax[e].y);
}

__global__ void add_kernel(const double2* __restrict__ a, long long n, double2* __restrict__ x) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < n) x[e] = make_double2(x[e].x + a[e].x, x[e].y + a[e].y);
}

namespace {

struct Vec {
    aim_plan* p;
    cudaStream_t s;
    long long n;
    double2* part;        // [kPartBlocks][kGmChunk]
    double2* dcoef;       // [3][kMaxBasis + 1] device coefficients: h1, h2, misc
    const GmresOps& ops;

    unsigned nb() const { return (unsigned)((n + 255) / 256); }
    int an_blocks() const { return (int)std::max(1LL, std::min<long long>(kAnBlocks, (n + kAnThreads - 1) / kAnThreads)); }
    void reduce(int nv, double2* out, bool acc, int nb = kGmBlocks) {
        gm_reduce_kernel<<<(nv + 7) / 8, 256, 0, s>>>(part, nb, nv, out, acc ? 1 : 0);
        note_launch("gmres_reduce");
    }
    void allreduce(double2* d, int nv) {
        if (ops.allreduce) ops.allreduce(d, nv, s);
    }
    // out[0..nv) = V^H w (device)
    void dots(const double2* V, int nv, const double2* w, double2* out) {
        for (int i0 = 0; i0 < nv; i0 += kGmChunk) {
            const int m = std::min(kGmChunk, nv - i0);
            mdot_kernel<4><<<kGmBlocks, kGmThreads, 0, s>>>(V + (size_t)i0 * n, n, n, m, w, part);
            note_launch("gmres_mdot");
            reduce(m, out + i0, false);
        }
        allreduce(out, nv);
    }
    // w -= V c, then out = V^H w
    void axpy_dots(const double2* V, int nv, const double2* c, double2* w, double2* out) {
        if (nv <= kGmChunk) {
            {
                static unsigned long long attr_mask = 0;   // the attribute is per device
                if (!(attr_mask >> (p->device & 63) & 1ULL)) {
                    AIM_CUDA(cudaFuncSetAttribute(axpy_dot_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  (int)(2 * (kGmChunk + 1) * kAdT * sizeof(double2))));
                    attr_mask |= 1ULL << (p->device & 63);
                }
                const size_t smem = 2 * (size_t)(nv + 1) * kAdT * sizeof(double2);
                axpy_dot_smem_kernel<<<kAdBlocks, kAdThreads, smem, s>>>(V, n, n, nv, c, w, part);
            }
            note_launch("gmres_axpy_dot");
            reduce(nv, out, false, kAdBlocks);
            allreduce(out, nv);
            return;
        }
        axpy(V, nv, c, w, nullptr);
        dots(V, nv, w, out);
    }
    // w -= V c (and ||w||^2 into *nrm2 when given)
    void axpy(const double2* V, int nv, const double2* c, double2* w, double2* nrm2) {
        for (int i0 = 0; i0 < nv; i0 += kGmChunk) {
            const int m = std::min(kGmChunk, nv - i0);
            const bool last = i0 + m >= nv;
            axpy_norm_kernel<<<an_blocks(), kAnThreads, 0, s>>>(V + (size_t)i0 * n, n, n, m, c + i0, w, part,
                                                                (last && nrm2) ? 1 : 0);
            note_launch("gmres_axpy_norm");
        }
        if (nrm2) {
            reduce(1, nrm2, false, an_blocks());
            allreduce(nrm2, 1);
        }
    }
    void norm2(const double2* w, double2* out) {
        dots(w, 1, w, out);
    }
    void scale(const double2* src, const double2* nrm2, double2* dst, double2* dst2 = nullptr) {
        gm_scale_kernel<<<nb(), 256, 0, s>>>(src, n, nrm2, dst, dst2);
        note_launch("gmres_scale");
    }
    void combine(const double2* V, int nv, const double2* y, double2* out, bool acc) {
        for (int i0 = 0; i0 < nv; i0 += kGmChunk) {
            const int m = std::min(kGmChunk, nv - i0);
            gm_combine_kernel<<<nb(), 256, 0, s>>>(V + (size_t)i0 * n, n, n, m, y + i0, out, (acc || i0) ? 1 : 0);
            note_launch("gmres_combine");
        }
    }
};

inline bool finite(cplx z) { return std::isfinite(z.real()) && std::isfinite(z.imag()); }

}  // namespace

int gmres(aim_plan* p, const double2* b, double2* x, int restart, double tol, int max_iters, int fixed_iters,
          int* iters_out, double* rel_out) {
    GmresOps ops;
    ops.n = p->N;
    ops.matvec = [p](const double2* in, double2* out, cudaStream_t st) { matvec(p, in, out, 1, st); };
    if (p->prec_on) ops.precond = [p](const double2* in, double2* out, cudaStream_t st) { apply_precond(p, in, out, st); };
    return gmres_core(p, ops, b, x, restart, tol, max_iters, fixed_iters, iters_out, rel_out);
}

// The solver with any operator on vectors of local length ops.n: `p` holds the
// workspace and the stream; ops.matvec applies A, ops.precond (optional) M^-1,
// ops.allreduce (optional) sums small device vectors over the ranks.
int gmres_core(aim_plan* p, const GmresOps& ops, const double2* b, double2* x, int restart, double tol,
               int max_iters, int fixed_iters, int* iters_out, double* rel_out) {
    if (restart < 1 || restart + 1 > kMaxBasis) throw Error(AIM_E_ARG, "restart must be in [1, 1023]");
    if (max_iters <= 0) max_iters = 20000;
    const long long n = ops.n;
    cudaStream_t s = p->stream;
    const bool pre = (bool)ops.precond;
    if (p->gm_restart < restart || p->gm_n != n || !p->gm_z) {
        p->release(p->gm_V);
        p->release(p->gm_w);
        p->release(p->gm_z);
        p->release(p->gm_part);
        p->gm_V = p->alloc<double2>((size_t)(restart + 1) * std::max(1LL, n));
        p->gm_w = p->alloc<double2>(std::max(1LL, n));
        p->gm_z = p->alloc<double2>(std::max(1LL, n));
        p->gm_part = p->alloc<double2>((size_t)kPartBlocks * kGmChunk + 3 * (kMaxBasis + 1));
        p->gm_restart = restart;
        p->gm_n = n;
    }
    if (!p->gm_host) AIM_CUDA(cudaMallocHost(&p->gm_host, sizeof(double2) * 3 * (kMaxBasis + 1)));
    double2* hbuf = p->gm_host;
    Vec g{p, s, n, p->gm_part, p->gm_part + (size_t)kPartBlocks * kGmChunk, ops};
    double2* dh1 = g.dcoef;
    // h1, h2 and ||w||^2 of an iteration are adjacent (one fetch):
    // [h1: cst][h2: cst][misc: [0] ||.||^2, [1..] y coefficients], cst = restart + 1
    const int cst = restart + 1;
    double2* dh2 = g.dcoef + cst;
    double2* dmisc = g.dcoef + 2 * cst;
    double2* V = p->gm_V;
    double2* w = p->gm_w;
    double2* z = p->gm_z;
    const int limit = fixed_iters > 0 ? fixed_iters : max_iters;
    p->gm_hist.clear();

    auto fetch = [&](const double2* d, int cnt, double2* h) {
        AIM_CUDA(cudaMemcpyAsync(h, d, sizeof(double2) * cnt, cudaMemcpyDeviceToHost, s));
    };
    auto sync = [&]() { AIM_CUDA(cudaStreamSynchronize(s)); };
    if (!p->gm_ev) AIM_CUDA(cudaEventCreateWithFlags(&p->gm_ev, cudaEventDisableTiming | cudaEventBlockingSync));
    // the product of basis vector j (v_j in V[j]; for the unpreconditioned
    // solve also in z, the product's fixed input)
    auto product = [&](int j) {
        if (pre) {
            ops.precond(V + (size_t)j * n, z, s);
            ops.matvec(z, w, s);
        } else {
            ops.matvec(z, w, s);
        }
    };

    AIM_CUDA(cudaMemsetAsync(x, 0, sizeof(double2) * n, s));
    g.norm2(b, dmisc);
    fetch(dmisc, 1, hbuf);
    sync();
    if (!std::isfinite(hbuf[0].x)) throw Error(AIM_E_BREAKDOWN, "GMRES: right-hand side is not finite");
    const double bnorm = std::sqrt(std::max(0.0, hbuf[0].x));
    if (!std::isfinite(bnorm)) throw Error(AIM_E_BREAKDOWN, "GMRES: right-hand side is not finite");
    if (bnorm == 0.0) {
        if (iters_out) *iters_out = 0;
        if (rel_out) *rel_out = 0.0;
        return AIM_OK;
    }
    // r0 = b (x0 = 0)
    // Unpreconditioned products read v_j from z, a copy written with it, so the
    // product's CUDA graph (keyed on its input and output pointers) is captured
    // once per solve instead of once per basis vector.
    double2* zin = pre ? nullptr : z;
    double beta = bnorm;
    g.scale(b, dmisc, V, zin);
    int total = 0;
    double rel = 1.0;
    std::vector<cplx> H((size_t)(restart + 1) * restart), gv(restart + 1), sn(restart);
    std::vector<double> cs(restart);
    auto Hij = [&](int i, int j) -> cplx& { return H[(size_t)i * restart + j]; };
    while (true) {
        std::fill(H.begin(), H.end(), cplx(0));
        std::fill(gv.begin(), gv.end(), cplx(0));
        gv[0] = beta;
        int jd = 0;
        bool stop = false;
        bool pending = false;   // the product of v_j is already enqueued
        for (int j = 0; j < restart; ++j) {
            if (!pending) product(j);
            pending = false;
            const int nv = j + 1;
            g.dots(V, nv, w, dh1);                 // pass 1
            g.axpy_dots(V, nv, dh1, w, dh2);       // pass 2
            g.axpy(V, nv, dh2, w, dmisc);          // pass 3 (+ ||w||^2)
            g.scale(w, dmisc, V + (size_t)(j + 1) * n, zin);
            fetch(dh1, 2 * cst + 1, hbuf);
            AIM_CUDA(cudaEventRecord(p->gm_ev, s));
            // v_{j+1} is complete on the device: enqueue its product before the
            // host works on the coefficients, so the GPU does not idle during
            // the Givens update (wasted once per solve if this iteration converges)
            if (j + 1 < restart && total + 1 < limit) {
                product(j + 1);
                pending = true;
            }
            AIM_CUDA(cudaEventSynchronize(p->gm_ev));
            for (int i = 0; i <= j; ++i) {
                Hij(i, j) = cplx(hbuf[i].x, hbuf[i].y) + cplx(hbuf[cst + i].x, hbuf[cst + i].y);
                if (!finite(Hij(i, j))) throw Error(AIM_E_BREAKDOWN, "GMRES: non-finite Arnoldi coefficient");
            }
            const double hn2 = hbuf[2 * cst].x;
            const double hn = std::isfinite(hn2) ? std::sqrt(std::max(0.0, hn2)) : hn2;
            if (!std::isfinite(hn)) throw Error(AIM_E_BREAKDOWN, "GMRES: non-finite Arnoldi norm");
            Hij(j + 1, j) = hn;
            for (int i = 0; i < j; ++i) {
                const cplx t = cs[i] * Hij(i, j) + sn[i] * Hij(i + 1, j);
                Hij(i + 1, j) = -std::conj(sn[i]) * Hij(i, j) + cs[i] * Hij(i + 1, j);
                Hij(i, j) = t;
            }
            const cplx a = Hij(j, j), bb = Hij(j + 1, j);
            double c;
            cplx sgv;
            if (std::abs(a) == 0.0) {
                c = 0.0;
                sgv = 1.0;
            } else {
                const double r = std::sqrt(std::norm(a) + std::norm(bb));
                c = std::abs(a) / r;
                sgv = (a / std::abs(a)) * std::conj(bb) / r;
            }
            cs[j] = c;
            sn[j] = sgv;
            Hij(j, j) = c * Hij(j, j) + sgv * Hij(j + 1, j);
            Hij(j + 1, j) = 0.0;
            gv[j + 1] = -std::conj(sgv) * gv[j];
            gv[j] = c * gv[j];
            ++total;
            jd = j + 1;
            const double est = std::abs(gv[j + 1]) / bnorm;
            p->gm_hist.push_back(est);
            if (total >= limit) { stop = true; break; }
            if (fixed_iters <= 0 && est <= tol) break;
            if (hn == 0) break;
        }
        // y = H^-1 g (upper triangular), x += M^-1 (V y)
        std::vector<cplx> yv(jd);
        for (int i = jd - 1; i >= 0; --i) {
            cplx t = gv[i];
            for (int q = i + 1; q < jd; ++q) t -= Hij(i, q) * yv[q];
            yv[i] = t / Hij(i, i);
            if (!finite(yv[i])) throw Error(AIM_E_BREAKDOWN, "GMRES: singular Hessenberg matrix");
        }
        if (jd) {
            for (int i = 0; i < jd; ++i) hbuf[i] = make_double2(yv[i].real(), yv[i].imag());
            AIM_CUDA(cudaMemcpyAsync(dmisc + 1, hbuf, sizeof(double2) * jd, cudaMemcpyHostToDevice, s));
            if (pre) {
                g.combine(V, jd, dmisc + 1, w, false);
                ops.precond(w, z, s);
                add_kernel<<<g.nb(), 256, 0, s>>>(z, n, x);
                note_launch("gmres_add");
            } else {
                g.combine(V, jd, dmisc + 1, x, true);
            }
        }
        // true residual r = b - A x into V[0]
        ops.matvec(x, w, s);
        residual_kernel<<<g.nb(), 256, 0, s>>>(b, w, n, V);
        note_launch("gmres_residual");
        g.norm2(V, dmisc);
        fetch(dmisc, 1, hbuf);
        sync();
        beta = std::isfinite(hbuf[0].x) ? std::sqrt(std::max(0.0, hbuf[0].x)) : hbuf[0].x;
        if (!std::isfinite(beta)) throw Error(AIM_E_BREAKDOWN, "GMRES: non-finite residual");
        rel = beta / bnorm;
        if (stop || (fixed_iters <= 0 && rel <= tol) || beta == 0.0) break;
        g.scale(V, dmisc, V, zin);
    }
    sync();
    if (iters_out) *iters_out = total;
    if (rel_out) *rel_out = rel;
    return rel <= tol ? AIM_OK : AIM_NOT_CONVERGED;
}

}  // namespace aim
