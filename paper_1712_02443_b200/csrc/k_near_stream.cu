// H6 near-field SpMV, single right-hand side, staged by TMA bulk copies and
// overlapped with the FFT passes (step (iv) of the AIM matvec, the sparse
// precorrection y += Z_near x, PAPER.md:551-554 eq. AIM_step4 / SURVEY
// section 8(a) H6).
//
// Idea: the C4 product is near (1.49 ms, HBM-bound at the copy roofline),
// projection, three FFT passes (0.9 ms, shared-memory / FP64 bound, HBM
// mostly idle) and interpolation.  The plain warp-per-row SpMV keeps its
// bytes in flight in registers, so it needs every warp slot of every SM;
// launched beside the FFT it only queues behind it.  Here the value, column
// and row-pointer streams of a chunk go through shared memory by
// cp.async.bulk (TMA), so a 4-warp CTA small enough to sit beside the
// persistent FFT CTA (x pass: 448 threads, 164 KB smem; fused y/z pass: 392
// threads, 184 KB) can stream part of the near matrix while the FFT
// computes; after the FFT a register-pipelined warp-per-row kernel takes the
// chunks that are left from the same atomic counter.
//
// Measured (C4, one RHS; tools/ovl_ab.py, profiles/ovl_ab_r02_c4.log):
// SLOWER, so it is opt-in (AIM_NEAR_OVL=1).  The thin CTA is latency-bound
// on the x gathers (a few rows in flight per SM, ~7 us per 10 KB chunk), and
// whenever the side CTAs land on an SM first the persistent FFT CTA waits
// for them; the chunk counter costs ~0.1 ms over near1 at full occupancy.
//
// Rows are cut into chunks of at most kNsCap entries (built once per plan).
// Each row is summed by one warp in exactly near1_kernel's order (lane l
// accumulates entries l, l + 32, l + 64, ... with the same fma sequence,
// then the xor butterfly), so the result is bit-identical to near1_kernel's
// whichever CTA takes the chunk.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <vector>

#include "aim_internal.cuh"
#include "cplx.cuh"

namespace aim {

namespace {

constexpr int kNsCap = 512;         // entries per chunk (smem: fits beside the 184 KB fused y/z CTA)
constexpr int kNsRows = 64;         // rows per chunk
constexpr int kNsPad = kNsCap + 4;  // + alignment slack of the 16-byte bulk copies
constexpr int kNsRowPad = kNsRows + 4;
constexpr int kNsStages = 2;
constexpr int kNsWarps = 4;
constexpr int kNsUnroll = 4;

__device__ __forceinline__ unsigned ns_smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void ns_mbar_init(uint64_t* m) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(ns_smem_u32(m)) : "memory");
}
__device__ __forceinline__ void ns_mbar_expect_tx(uint64_t* m, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(ns_smem_u32(m)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void ns_mbar_wait(uint64_t* m, unsigned phase) {
    asm volatile(
        "{\n .reg .pred P;\n NSW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra NSW_%=;\n}\n" ::"r"(
            ns_smem_u32(m)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void ns_bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* m) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     ns_smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(ns_smem_u32(m))
                 : "memory");
}

template <class C>
constexpr size_t ns_smem_bytes() {
    return (size_t)kNsStages * (kNsPad * (sizeof(C) + sizeof(int32_t)) + kNsRowPad * sizeof(int64_t));
}

// Chunk c: rows crow[c] .. crow[c+1]-1 (<= kNsRows), entries cent[c] ..
// cent[c+1]-1 (<= kNsCap).  Per stage the bulk copies bring the chunk's
// values, columns and row pointers; val/col/rowp are padded by >= 16 bytes
// past their ends (the copies round up to 16 bytes).
template <class C>
__global__ void __launch_bounds__(32 * kNsWarps, 16) near_stream_kernel(
    const int64_t* __restrict__ rowp, const int32_t* __restrict__ col, const C* __restrict__ val,
    const int32_t* __restrict__ crow, const int64_t* __restrict__ cent, int nchunks, int stop,
    unsigned* __restrict__ ctr, const C* __restrict__ x, C* __restrict__ y) {
    extern __shared__ __align__(128) unsigned char ns_smem[];
    C* vb = (C*)ns_smem;                                                              // [S][kNsPad]
    int32_t* cb = (int32_t*)(ns_smem + (size_t)kNsStages * kNsPad * sizeof(C));       // [S][kNsPad]
    int64_t* rb = (int64_t*)(ns_smem + (size_t)kNsStages * kNsPad * (sizeof(C) + 4));  // [S][kNsRowPad]
    __shared__ __align__(8) uint64_t mbar[kNsStages];
    __shared__ int cid[kNsStages], rbase[kNsStages], rend[kNsStages];
    __shared__ long long vbase[kNsStages], cbase[kNsStages];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    // thread 0: take the next chunk from the counter and start its copies
    // (no chunks taken once one at or past `stop` was: the rest is left to the
    // launch after the FFT, so this one never holds the SMs for long)
    __shared__ int stopped;
    auto issue = [&](int st) {
        const int c = stopped ? INT_MAX : (int)atomicAdd(ctr, 1u);
        if (c >= stop) stopped = 1;
        cid[st] = c;
        if (c < nchunks) {
            constexpr long long AV = 16 / sizeof(C);
            const int r0 = crow[c], r1 = crow[c + 1];
            const long long e0 = cent[c], e1 = cent[c + 1];
            const long long v0 = e0 & ~(AV - 1), c0 = e0 & ~3LL;
            const int q0 = r0 & ~1;
            const unsigned bv = (unsigned)max(16LL, ((e1 - v0) * (long long)sizeof(C) + 15) & ~15LL);
            const unsigned bc = (unsigned)max(16LL, ((e1 - c0) * 4 + 15) & ~15LL);
            const unsigned br = (unsigned)(((r1 + 1 - q0) * 8 + 15) & ~15);
            vbase[st] = v0;
            cbase[st] = c0;
            rbase[st] = q0;
            rend[st] = r1;
            ns_mbar_expect_tx(&mbar[st], bv + bc + br);
            ns_bulk_g2s(vb + st * kNsPad, val + v0, bv, &mbar[st]);
            ns_bulk_g2s(cb + st * kNsPad, col + c0, bc, &mbar[st]);
            ns_bulk_g2s(rb + st * kNsRowPad, rowp + q0, br, &mbar[st]);
        }
    };
    if (threadIdx.x == 0) {
        stopped = 0;
        for (int st = 0; st < kNsStages; ++st) ns_mbar_init(&mbar[st]);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        for (int st = 0; st < kNsStages; ++st) issue(st);
    }
    __syncthreads();
    // Chunks come off the counter in increasing order, so the first stage
    // found past the end has no copy in flight behind it.
    for (int it = 0;; ++it) {
        const int st = it % kNsStages;
        const int c = cid[st];
        if (c >= nchunks) break;
        ns_mbar_wait(&mbar[st], (unsigned)(it / kNsStages) & 1u);
        const C* v = vb + st * kNsPad - vbase[st];       // v[e], e in the chunk's entry range
        const int32_t* cc = cb + st * kNsPad - cbase[st];
        const int64_t* rp = rb + st * kNsRowPad - rbase[st];
        const int r1 = rend[st];
        for (int r = crow[c] + warp; r < r1; r += kNsWarps) {
            const long long e0 = rp[r], e1 = rp[r + 1];
            C acc = mkc<C>(0, 0);
            for (long long b = e0 + lane; b < e1; b += 32 * kNsUnroll) {
                C xv[kNsUnroll];
                int n[kNsUnroll];
#pragma unroll
                for (int u = 0; u < kNsUnroll; ++u) {
                    const long long e = b + 32 * u;
                    n[u] = e < e1 ? cc[e] : -1;
                }
#pragma unroll
                for (int u = 0; u < kNsUnroll; ++u) xv[u] = n[u] >= 0 ? __ldg(&x[n[u]]) : mkc<C>(0, 0);
#pragma unroll
                for (int u = 0; u < kNsUnroll; ++u) {
                    const long long e = b + 32 * u;
                    const C z = n[u] >= 0 ? v[e] : mkc<C>(0, 0);
                    acc.x = fma(z.x, xv[u].x, acc.x); acc.x = fma(-z.y, xv[u].y, acc.x);
                    acc.y = fma(z.x, xv[u].y, acc.y); acc.y = fma(z.y, xv[u].x, acc.y);
                }
            }
#pragma unroll
            for (int off = 16; off; off >>= 1) {
                const C t = shfl_xor2(acc, off);
                acc.x += t.x; acc.y += t.y;
            }
            if (lane == 0) y[r] = acc;
        }
        __syncthreads();                 // every warp is done with stage st
        if (threadIdx.x == 0) issue(st);
    }
}

// The rows left after the FFT: near1_kernel's register-pipelined warp per
// row at full occupancy, rows taken chunk by chunk from the same counter
// (lane 0 takes a chunk for its warp).
template <class C>
__global__ void __launch_bounds__(256) near_dyn_kernel(const int64_t* __restrict__ rowp,
                                                       const int32_t* __restrict__ col, const C* __restrict__ val,
                                                       const int32_t* __restrict__ crow, int nchunks,
                                                       unsigned* __restrict__ ctr, const C* __restrict__ x,
                                                       C* __restrict__ y) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        int c = 0;
        if (lane == 0) c = (int)atomicAdd(ctr, 1u);
        c = __shfl_sync(0xffffffffu, c, 0);
        if (c >= nchunks) return;
        const int r1 = crow[c + 1];
        for (int m = crow[c]; m < r1; ++m) {
            const long long e0 = rowp[m], e1 = rowp[m + 1];
            C acc = mkc<C>(0, 0);
            for (long long b = e0 + lane; b < e1; b += 128) {
                C z[4], xv[4];
                int n[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const long long e = b + 32 * u;
                    const bool v = e < e1;
                    z[u] = v ? __ldcs(&val[e]) : mkc<C>(0, 0);
                    n[u] = v ? __ldcs(&col[e]) : -1;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) xv[u] = n[u] >= 0 ? __ldg(&x[n[u]]) : mkc<C>(0, 0);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    acc.x = fma(z[u].x, xv[u].x, acc.x); acc.x = fma(-z[u].y, xv[u].y, acc.x);
                    acc.y = fma(z[u].x, xv[u].y, acc.y); acc.y = fma(z[u].y, xv[u].x, acc.y);
                }
            }
#pragma unroll
            for (int off = 16; off; off >>= 1) {
                const C t = shfl_xor2(acc, off);
                acc.x += t.x; acc.y += t.y;
            }
            if (lane == 0) y[m] = acc;
        }
    }
}

int sm_count_ns() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        AIM_CUDA(cudaGetDevice(&dev));
        AIM_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    }
    return n;
}

template <class C>
void ensure_ns_attr(int dev) {
    static unsigned long long mask = 0;  // per device
    if (mask >> (dev & 63) & 1ULL) return;
    AIM_CUDA(cudaFuncSetAttribute(near_stream_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)ns_smem_bytes<C>()));
    // keep the SM in its largest shared-memory configuration, so the CTA can
    // sit beside the FFT's 164-176 KB CTAs without a carveout change
    AIM_CUDA(cudaFuncSetAttribute(near_stream_kernel<C>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    mask |= 1ULL << (dev & 63);
}

}  // namespace

// AIM_NEAR_OVL=1 turns the overlap on (measured slower, see the header; off by
// default); the number of near CTAs per SM beside the FFT is AIM_NEAR_OVL_A
// (default 1, 0 = none), their share of the chunks AIM_NEAR_OVL_F.
int near_overlap_mode() {
    const char* e = getenv("AIM_NEAR_OVL");
    return (e && e[0] == '1') ? 1 : 0;
}

// AIM_NEAR_PRIO=1: near1 (128-thread CTAs) on the side stream beside the FFT
// passes, which run on a high-priority stream (k_matvec.cu matvec_body).
int near_prio_mode() {
    const char* e = getenv("AIM_NEAR_PRIO");
    return (e && e[0] == '1') ? 1 : 0;
}

// keep every SM in its largest shared-memory configuration (both overlap modes)
int smem_carveout_max() {
    const char* e = getenv("AIM_NEAR_CARVE");   // A/B: 0 = leave the FFT kernels' carveout alone
    if (e && e[0] == '0') return 0;
    return near_overlap_mode() || near_prio_mode();
}

static int near_overlap_ctas() {
    const char* e = getenv("AIM_NEAR_OVL_A");
    const int a = e ? atoi(e) : 1;
    return std::max(0, std::min(a, 4));
}

// Build the chunk table once (host pass over the row pointers).  Returns
// false when the streamed kernel does not apply (a row longer than a chunk).
bool near_stream_ready(aim_plan* p, cudaStream_t s) {
    if (p->ns_state) return p->ns_state > 0;
    p->ns_state = -1;
    if (p->N <= 0 || p->nnzN <= 0 || !p->nrow || !p->ncol_padded) return false;
    std::vector<int64_t> rowp(p->N + 1);
    AIM_CUDA(cudaMemcpyAsync(rowp.data(), p->nrow, sizeof(int64_t) * (p->N + 1), cudaMemcpyDeviceToHost, s));
    AIM_CUDA(cudaStreamSynchronize(s));
    std::vector<int32_t> crow(1, 0);
    std::vector<int64_t> cent(1, 0);
    for (long long r = 0; r < p->N; ++r) {
        if (rowp[r + 1] - rowp[r] > kNsCap) return false;
        if (rowp[r + 1] - rowp[crow.back()] > kNsCap || r - crow.back() >= kNsRows) {
            crow.push_back((int32_t)r);
            cent.push_back(rowp[r]);
        }
    }
    crow.push_back((int32_t)p->N);
    cent.push_back(rowp[p->N]);
    p->ns_count = (int)crow.size() - 1;
    p->ns_crow = p->alloc<int32_t>(crow.size());
    p->ns_cent = p->alloc<int64_t>(cent.size());
    p->ns_ctr = p->alloc<unsigned>(1);
    h2d(p->ns_crow, crow.data(), sizeof(int32_t) * crow.size(), s);
    h2d(p->ns_cent, cent.data(), sizeof(int64_t) * cent.size(), s);
    p->ns_state = 1;
    return true;
}

void near_stream_reset(aim_plan* p, cudaStream_t s) {
    AIM_CUDA(cudaMemsetAsync(p->ns_ctr, 0, sizeof(unsigned), s));
}

// ctas_per_sm > 0: the TMA-staged kernel, that many CTAs per SM (beside the
// FFT); 0: the register-pipelined warp-per-row kernel at full occupancy.
void launch_near_stream(aim_plan* p, const void* x, void* y, int ctas_per_sm, cudaStream_t s) {
    int dev = 0;
    AIM_CUDA(cudaGetDevice(&dev));
    const bool c64 = p->prec == AIM_C64;
    if (ctas_per_sm <= 0) {
        int per = 0;
        if (c64)
            AIM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, near_dyn_kernel<float2>, 256, 0));
        else
            AIM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, near_dyn_kernel<double2>, 256, 0));
        const unsigned grid = (unsigned)std::min<long long>((long long)std::max(1, per) * sm_count_ns(),
                                                            ((long long)p->ns_count + 7) / 8);
        if (c64)
            near_dyn_kernel<float2><<<grid, 256, 0, s>>>(p->nrow, p->ncol, p->nval32, p->ns_crow, p->ns_count,
                                                         p->ns_ctr, (const float2*)x, (float2*)y);
        else
            near_dyn_kernel<double2><<<grid, 256, 0, s>>>(p->nrow, p->ncol, p->nval, p->ns_crow, p->ns_count,
                                                          p->ns_ctr, (const double2*)x, (double2*)y);
        note_launch("near_dyn");
        return;
    }
    const unsigned grid = (unsigned)std::min<long long>((long long)ctas_per_sm * sm_count_ns(), p->ns_count);
    // share of the chunks the launch beside the FFT may take (AIM_NEAR_OVL_F)
    const char* ef = getenv("AIM_NEAR_OVL_F");
    const double frac = ef ? atof(ef) : 0.25;
    const int stop = (int)std::min<double>(p->ns_count, std::max(0.0, frac) * p->ns_count);
    if (c64) {
        ensure_ns_attr<float2>(dev);
        near_stream_kernel<float2><<<grid, 32 * kNsWarps, ns_smem_bytes<float2>(), s>>>(
            p->nrow, p->ncol, p->nval32, p->ns_crow, p->ns_cent, p->ns_count, stop, p->ns_ctr, (const float2*)x, (float2*)y);
    } else {
        ensure_ns_attr<double2>(dev);
        near_stream_kernel<double2><<<grid, 32 * kNsWarps, ns_smem_bytes<double2>(), s>>>(
            p->nrow, p->ncol, p->nval, p->ns_crow, p->ns_cent, p->ns_count, stop, p->ns_ctr, (const double2*)x, (double2*)y);
    }
    note_launch("near_stream");
}

int near_overlap_ctas_per_sm() { return near_overlap_ctas(); }

}  // namespace aim
