// Per-matvec kernels of y = Z_eq x:
//   H1 projection  Q^psi[u,r] = sum_{n in col(u)} w^psi_{n,u} x[n,r]
//      deterministic gather over the grid-node-sorted CSR, warp per node,
//      lanes over (entry group, rhs), fixed-order shuffle reduction;
//   H2-H4 convolution Phi = H Q by five Stockham passes (k_fft.cu):
//      x fwd (pad) -> y fwd (pad) -> z turnaround (pad, x G^, prune) ->
//      y inv (prune) -> x inv (prune)
//   H5+H6 interpolation y = j k eta0 [sum_xyz P^T Phi - k^-2 P_phi^T Phi_phi]
//       fused with the precorrected near-field SpMV
//      y += Z_corr x: warp per RWG row, one y write.
#include <math.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "aim_internal.cuh"
#include "cplx.cuh"

namespace aim {

static inline unsigned nblk(long long n, int t) { return (unsigned)((n + t - 1) / t); }

#ifndef AIM_GATHER_UNROLL
#define AIM_GATHER_UNROLL 2
#endif
#ifndef AIM_GATHER_RPL16
#define AIM_GATHER_RPL16 1
#endif
constexpr int kGatherUnroll = AIM_GATHER_UNROLL;   // gather steps in flight per lane
#ifndef AIM_P1_UNROLL
#define AIM_P1_UNROLL 4
#endif
constexpr int kP1Unroll = AIM_P1_UNROLL;           // single-RHS projection: entries in flight per lane


// Lane layout of the gather kernels: LPE lanes share one CSR entry and each
// holds RPL right-hand sides (r = r0 + sub + q*LPE), so a warp consumes
// G = 32/LPE entries per step; the LPE lanes of a group read LPE*16
// contiguous bytes per load.  Entries are staged 32 at a time: lane e loads
// entry e's index / value (coalesced), then broadcasts it with shuffles.
template <int LPE, int RPL>
struct Lanes {
    static constexpr int G = 32 / LPE;
    static constexpr int RC = LPE * RPL;
    int lane, grp, sub;
    __device__ __forceinline__ Lanes() {
        lane = threadIdx.x & 31;
        grp = lane / LPE;
        sub = lane % LPE;
    }
};

// ------------------------------------------------------------ H1 projection
// Q^psi[u,r] = sum_{n in col(u)} w^psi_{n,u} x[n,r]; warp per grid node.
// The weights are read in CSR order (Wc, pn: coalesced streams), not gathered.
template <int M, int LPE, int RPL, class C>
__global__ void __launch_bounds__(256) project_kernel(const int32_t* __restrict__ prow,
                                                      const int32_t* __restrict__ pn,
                                                      const Real<C>* __restrict__ Wc, const C* __restrict__ x,
                                                      long long Ng, int R, C* __restrict__ Q) {
    using L = Lanes<LPE, RPL>;
    const long long g = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / 32;
    if (g >= Ng) return;
    const L ln;
    const int e0 = prow[g], e1 = prow[g + 1];
    const C* W2 = reinterpret_cast<const C*>(Wc);
    for (int r0 = 0; r0 < R; r0 += L::RC) {
        C a[4][RPL];
#pragma unroll
        for (int q = 0; q < RPL; ++q)
            for (int c = 0; c < 4; ++c) a[c][q] = mkc<C>(0, 0);
        for (int b = e0; b < e1; b += 32) {
            const int cnt = min(32, e1 - b);
            int n_l = 0;
            C w01 = mkc<C>(0, 0), w23 = w01;
            if (ln.lane < cnt) {
                n_l = __ldcs(&pn[b + ln.lane]);
                w01 = __ldcs(W2 + 2 * (long long)(b + ln.lane));
                w23 = __ldcs(W2 + 2 * (long long)(b + ln.lane) + 1);
            }
#pragma unroll kGatherUnroll
            for (int t = ln.grp; t < 32; t += L::G) {
                int n;
                Real<C> w[4];
                if (LPE == 1) {
                    n = n_l; w[0] = w01.x; w[1] = w01.y; w[2] = w23.x; w[3] = w23.y;
                } else {
                    n = __shfl_sync(0xffffffffu, n_l, t);
                    w[0] = __shfl_sync(0xffffffffu, w01.x, t); w[1] = __shfl_sync(0xffffffffu, w01.y, t);
                    w[2] = __shfl_sync(0xffffffffu, w23.x, t); w[3] = __shfl_sync(0xffffffffu, w23.y, t);
                }
                if (t < cnt) {
                    const C* xr = x + (long long)n * R + r0 + ln.sub;
#pragma unroll
                    for (int q = 0; q < RPL; ++q) {
                        if (r0 + ln.sub + q * LPE < R) {
                            const C xv = __ldg(xr + q * LPE);
#pragma unroll
                            for (int c = 0; c < 4; ++c) {
                                a[c][q].x = fma(w[c], xv.x, a[c][q].x);
                                a[c][q].y = fma(w[c], xv.y, a[c][q].y);
                            }
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int off = LPE; off < 32; off <<= 1)
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
                for (int q = 0; q < RPL; ++q) {
                    const C t = shfl_xor2(a[c][q], off);
                    a[c][q].x += t.x; a[c][q].y += t.y;
                }
        if (ln.grp == 0) {
#pragma unroll
            for (int q = 0; q < RPL; ++q) {
                const int rr = r0 + ln.sub + q * LPE;
                if (rr < R)
#pragma unroll
                    for (int c = 0; c < 4; ++c) __stcs(&Q[((long long)c * Ng + g) * R + rr], a[c][q]);
            }
        }
    }
}

// Single right-hand side (GMRES products): G lanes per grid node, 32/G nodes
// per warp, each lane strides over the node's entries (fixed order), group
// reduction by shuffles; a node's 4 components are written by its first lane.
template <int G, class C>
__global__ void __launch_bounds__(256) project1_kernel(const int32_t* __restrict__ prow,
                                                       const int32_t* __restrict__ pn,
                                                       const Real<C>* __restrict__ Wc, const C* __restrict__ x,
                                                       long long Ng, C* __restrict__ Q) {
    const long long gid = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / G;
    const int sub = threadIdx.x % G;
    const bool live = gid < Ng;
    const int e0 = live ? prow[gid] : 0, e1 = live ? prow[gid + 1] : 0;
    const C* W2 = reinterpret_cast<const C*>(Wc);
    C a[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) a[c] = mkc<C>(0, 0);
#pragma unroll kP1Unroll
    for (int e = e0 + sub; e < e1; e += G) {
        const int n = __ldcs(&pn[e]);
        const C w01 = __ldcs(W2 + 2 * (long long)e), w23 = __ldcs(W2 + 2 * (long long)e + 1);
        const C xv = __ldg(&x[n]);
        a[0].x = fma(w01.x, xv.x, a[0].x); a[0].y = fma(w01.x, xv.y, a[0].y);
        a[1].x = fma(w01.y, xv.x, a[1].x); a[1].y = fma(w01.y, xv.y, a[1].y);
        a[2].x = fma(w23.x, xv.x, a[2].x); a[2].y = fma(w23.x, xv.y, a[2].y);
        a[3].x = fma(w23.y, xv.x, a[3].x); a[3].y = fma(w23.y, xv.y, a[3].y);
    }
#pragma unroll
    for (int off = 1; off < G; off <<= 1)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const C t = shfl_xor2(a[c], off);
            a[c].x += t.x; a[c].y += t.y;
        }
    if (live && sub == 0)
#pragma unroll
        for (int c = 0; c < 4; ++c) __stcs(&Q[(long long)c * Ng + gid], a[c]);
}

// (LPE, RPL) per RHS count.  NEAR: 4 RHS per lane (instruction-bound SpMV);
// GATHER (projection / interpolation): one RHS per lane (latency-bound).
#define AIM_LANE_DISPATCH_NEAR(R, CALL)                \
    if (R == 1) { CALL(1, 1); }                        \
    else if (R == 2) { CALL(1, 2); }                   \
    else if (R <= 4) { CALL(1, 4); }                   \
    else if (R <= 8) { CALL(2, 4); }                   \
    else if (R <= 16) { CALL(4, 4); }                  \
    else { CALL(8, 4); }
#define AIM_LANE_DISPATCH_GATHER(R, CALL)              \
    if (R == 1) { CALL(1, 1); }                        \
    else if (R == 2) { CALL(2, 1); }                   \
    else if (R <= 4) { CALL(4, 1); }                   \
    else if (R <= 8) { CALL(8, 1); }                   \
    else if (R <= 16) { CALL(16 / AIM_GATHER_RPL16, AIM_GATHER_RPL16); } \
    else { CALL(32, 1); }

template <class C>
static void launch_project_t(const aim_plan* p, const C* x, C* Q, int R, cudaStream_t s) {
    const unsigned grid = nblk(p->Ng * 32, 256);
    const Real<C>* W = (const Real<C>*)(sizeof(C) == 16 ? (const void*)p->Wc : (const void*)p->Wc32);
    if (R == 1) {
        // lanes per node ~ entries per node / 4 (power of two in [4, 32])
        const double per = p->Ng ? (double)p->nnzP / (double)p->Ng : 1.0;
#ifndef AIM_P1_DIV
#define AIM_P1_DIV 8
#endif
        const double pl = per / AIM_P1_DIV;   // entries per lane ~ AIM_P1_DIV
        const int G = pl > 24 ? 32 : pl > 12 ? 16 : pl > 6 ? 8 : 4;
#define P1(GG) project1_kernel<GG, C><<<nblk(p->Ng * GG, 256), 256, 0, s>>>(p->prow, p->pn, W, x, p->Ng, Q)
        if (G == 32) P1(32);
        else if (G == 16) P1(16);
        else if (G == 8) P1(8);
        else P1(4);
#undef P1
        return;
    }
#define PJ_CALL(LPE, RPL) project_kernel<MM, LPE, RPL, C><<<grid, 256, 0, s>>>(p->prow, p->pn, W, x, p->Ng, R, Q)
#define PJ_M(MMV)                                   \
    if (p->M == MMV) {                              \
        constexpr int MM = MMV;                     \
        AIM_LANE_DISPATCH_GATHER(R, PJ_CALL)        \
        return;                                     \
    }
    PJ_M(1) PJ_M(2) PJ_M(3) PJ_M(4) PJ_M(5) PJ_M(6)
#undef PJ_M
#undef PJ_CALL
    throw Error(AIM_E_ARG, "unsupported M");
}

void launch_project(const aim_plan* p, const void* x, void* Q, int R, cudaStream_t s) {
    if (p->cp_on && R == 1) {   // repetition-compressed templates (NEXT-3, k_compress.cu)
        launch_project_cmp(p, x, Q, s);
        return;
    }
    if (p->prec == AIM_C64) launch_project_t(p, (const float2*)x, (float2*)Q, R, s);
    else launch_project_t(p, (const double2*)x, (double2*)Q, R, s);
    note_launch("project");
}

// ------------------------------------------------------ H5 interpolation
// y[m,r] (+)= j k eta0 [sum_xyz sum_u w_{m,u} Phi[u,r] - k^-2 sum_u w^phi_{m,u} Phi^phi[u,r]]
// Warp per RWG row: lane u loads w_{m,u} (contiguous) and its node index, then
// the rhs lanes gather the stencil's potentials (weights broadcast by shuffles).
template <int M, int LPE, int RPL, class C>
__global__ void __launch_bounds__(256) interp_kernel(const C* __restrict__ Phi, const Real<C>* __restrict__ W,
                                                     const int32_t* __restrict__ node0, long long Ng, int Ny, int Nz,
                                                     long long N, int R, double keta, double ik2, int accumulate,
                                                     C* __restrict__ y) {
    constexpr int M1 = M + 1, S = M1 * M1 * M1;
    using L = Lanes<LPE, RPL>;
    const long long m = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / 32;
    if (m >= N) return;
    const L ln;
    const long long g0 = node0[m];
    const C* W2 = reinterpret_cast<const C*>(W) + 2 * m * S;
    for (int r0 = 0; r0 < R; r0 += L::RC) {
        C aA[RPL], aP[RPL];
#pragma unroll
        for (int q = 0; q < RPL; ++q) aA[q] = aP[q] = mkc<C>(0, 0);
        for (int ub = 0; ub < S; ub += 32) {
            const int u_l = ub + ln.lane;
            const int cnt = min(32, S - ub);
            C w01 = mkc<C>(0, 0), w23 = w01;
            int g_l = 0;
            if (ln.lane < cnt) {
                w01 = __ldcs(W2 + 2 * u_l);
                w23 = __ldcs(W2 + 2 * u_l + 1);
                const int ui = u_l / (M1 * M1), uj = (u_l / M1) % M1, uk = u_l % M1;
                g_l = (int)(g0 + ((long long)ui * Ny + uj) * Nz + uk);
            }
#pragma unroll kGatherUnroll
            for (int t = ln.grp; t < 32; t += L::G) {
                int g;
                Real<C> w[4];
                if (LPE == 1) {
                    g = g_l; w[0] = w01.x; w[1] = w01.y; w[2] = w23.x; w[3] = w23.y;
                } else {
                    g = __shfl_sync(0xffffffffu, g_l, t);
                    w[0] = __shfl_sync(0xffffffffu, w01.x, t); w[1] = __shfl_sync(0xffffffffu, w01.y, t);
                    w[2] = __shfl_sync(0xffffffffu, w23.x, t); w[3] = __shfl_sync(0xffffffffu, w23.y, t);
                }
                if (t < cnt) {
#pragma unroll
                    for (int q = 0; q < RPL; ++q) {
                        const int rr = r0 + ln.sub + q * LPE;
                        if (rr < R) {
                            const C f0 = __ldg(&Phi[(0 * Ng + g) * R + rr]);
                            const C f1 = __ldg(&Phi[(1 * Ng + g) * R + rr]);
                            const C f2 = __ldg(&Phi[(2 * Ng + g) * R + rr]);
                            const C f3 = __ldg(&Phi[(3 * Ng + g) * R + rr]);
                            aA[q].x = fma(w[0], f0.x, aA[q].x); aA[q].y = fma(w[0], f0.y, aA[q].y);
                            aA[q].x = fma(w[1], f1.x, aA[q].x); aA[q].y = fma(w[1], f1.y, aA[q].y);
                            aA[q].x = fma(w[2], f2.x, aA[q].x); aA[q].y = fma(w[2], f2.y, aA[q].y);
                            aP[q].x = fma(w[3], f3.x, aP[q].x); aP[q].y = fma(w[3], f3.y, aP[q].y);
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
            // far = j k eta0 (aA - aP / k^2)
            const C f = mkc<C>(aA[q].x - aP[q].x * (Real<C>)ik2, aA[q].y - aP[q].y * (Real<C>)ik2);
            C tot = mkc<C>(-(Real<C>)keta * f.y, (Real<C>)keta * f.x);
#pragma unroll
            for (int off = LPE; off < 32; off <<= 1) {
                const C t = shfl_xor2(tot, off);
                tot.x += t.x; tot.y += t.y;
            }
            const int rr = r0 + ln.sub + q * LPE;
            if (ln.grp == 0 && rr < R) {
                if (accumulate) {
                    const C o = y[m * R + rr];
                    tot.x += o.x; tot.y += o.y;
                }
                y[m * R + rr] = tot;
            }
        }
    }
}

// Single right-hand side: warp per RWG row, lane u holds stencil entries
// u, u + 32, ... (K = ceil(S/32) of them): all weights, then all 4K potential
// gathers are issued before the FMAs; fixed order => deterministic.
template <int M, int RW, class C>
__global__ void __launch_bounds__(256) interp1_kernel(const C* __restrict__ Phi, const Real<C>* __restrict__ W,
                                                      const int32_t* __restrict__ node0, long long Ng, int Ny, int Nz,
                                                      long long N, double keta, double ik2, int accumulate,
                                                      const int32_t* __restrict__ wrow, C* __restrict__ y) {
    // RW rows per warp: every row's weights and node index are requested
    // before any row's potential gathers, which are all in flight together
    constexpr int M1 = M + 1, S = M1 * M1 * M1, K = (S + 31) / 32;
    const long long m0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / 32 * RW;
    if (m0 >= N) return;
    const int lane = threadIdx.x & 31;
    long long g0[RW];
#pragma unroll
    for (int q = 0; q < RW; ++q) g0[q] = m0 + q < N ? (long long)node0[m0 + q] : -1;
    C w01[RW][K], w23[RW][K];
#pragma unroll
    for (int q = 0; q < RW; ++q) {
        // wrow (repetition-compressed plans): the group representative's weight row
        const long long wr = wrow && g0[q] >= 0 ? (long long)__ldg(&wrow[m0 + q]) : m0 + q;
        const C* W2 = reinterpret_cast<const C*>(W) + 2 * wr * S;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int u = lane + 32 * k;
            const bool v = u < S && g0[q] >= 0;
            if constexpr (sizeof(C) == 16) {
                // the four weights of entry u in one 256-bit load (sm_100 LDG.E.256): half
                // the L1 wavefronts of two 128-bit loads
                double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
                if (v)
                    asm("ld.global.nc.L1::no_allocate.v4.f64 {%0, %1, %2, %3}, [%4];\n"
                                 : "=d"(a0), "=d"(a1), "=d"(a2), "=d"(a3)
                                 : "l"(W2 + 2 * u));
                w01[q][k] = mkc<C>(a0, a1);
                w23[q][k] = mkc<C>(a2, a3);
            } else {
                w01[q][k] = v ? __ldcs(W2 + 2 * u) : mkc<C>(0, 0);
                w23[q][k] = v ? __ldcs(W2 + 2 * u + 1) : mkc<C>(0, 0);
            }
        }
    }
    C f[RW][K][4];
#pragma unroll
    for (int q = 0; q < RW; ++q)
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int u = lane + 32 * k;
            const int ui = u / (M1 * M1), uj = (u / M1) % M1, uk = u % M1;
            const bool v = u < S && g0[q] >= 0;
            const long long g = g0[q] + ((long long)ui * Ny + uj) * Nz + uk;
#pragma unroll
            for (int c = 0; c < 4; ++c) f[q][k][c] = v ? __ldg(&Phi[c * Ng + g]) : mkc<C>(0, 0);
        }
#pragma unroll
    for (int q = 0; q < RW; ++q) {
        C aA = mkc<C>(0, 0), aP = mkc<C>(0, 0);
#pragma unroll
        for (int k = 0; k < K; ++k) {
            aA.x = fma(w01[q][k].x, f[q][k][0].x, aA.x); aA.y = fma(w01[q][k].x, f[q][k][0].y, aA.y);
            aA.x = fma(w01[q][k].y, f[q][k][1].x, aA.x); aA.y = fma(w01[q][k].y, f[q][k][1].y, aA.y);
            aA.x = fma(w23[q][k].x, f[q][k][2].x, aA.x); aA.y = fma(w23[q][k].x, f[q][k][2].y, aA.y);
            aP.x = fma(w23[q][k].y, f[q][k][3].x, aP.x); aP.y = fma(w23[q][k].y, f[q][k][3].y, aP.y);
        }
        // far = j k eta0 (aA - aP / k^2)
        const C fr = mkc<C>(aA.x - aP.x * (Real<C>)ik2, aA.y - aP.y * (Real<C>)ik2);
        C tot = mkc<C>(-(Real<C>)keta * fr.y, (Real<C>)keta * fr.x);
#pragma unroll
        for (int off = 16; off; off >>= 1) {
            const C t = shfl_xor2(tot, off);
            tot.x += t.x; tot.y += t.y;
        }
        if (lane == 0 && g0[q] >= 0) {
            if (accumulate) {
                const C o = y[m0 + q];
                tot.x += o.x; tot.y += o.y;
            }
            y[m0 + q] = tot;
        }
    }
}

// ------------------------------------------------------- H6 near SpMV
// y[m,r] = sum_{n in near(m)} Z_corr[m,n] x[n,r]; warp per row, entries
// staged 32 at a time (values streamed past L1), fixed-order reduction.
template <int LPE, int RPL, class C>
__global__ void __launch_bounds__(256) near_kernel(const int64_t* __restrict__ rowp, const int32_t* __restrict__ col,
                                                   const C* __restrict__ val, const C* __restrict__ x,
                                                   long long N, int R, C* __restrict__ y) {
    using L = Lanes<LPE, RPL>;
    const long long m = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / 32;
    if (m >= N) return;
    const L ln;
    const long long e0 = rowp[m], e1 = rowp[m + 1];
    for (int r0 = 0; r0 < R; r0 += L::RC) {
        C acc[RPL];
#pragma unroll
        for (int q = 0; q < RPL; ++q) acc[q] = mkc<C>(0, 0);
        for (long long b = e0; b < e1; b += 32) {
            const int cnt = (int)min(32LL, e1 - b);
            C z_l = mkc<C>(0, 0);
            int n_l = 0;
            if (ln.lane < cnt) {
                z_l = __ldcs(&val[b + ln.lane]);
                n_l = __ldcs(&col[b + ln.lane]);
            }
#pragma unroll 4
            for (int t = ln.grp; t < 32; t += L::G) {
                int n;
                Real<C> zx, zy;
                if (LPE == 1) {
                    n = n_l; zx = z_l.x; zy = z_l.y;
                } else {
                    n = __shfl_sync(0xffffffffu, n_l, t);
                    zx = __shfl_sync(0xffffffffu, z_l.x, t);
                    zy = __shfl_sync(0xffffffffu, z_l.y, t);
                }
                if (t < cnt) {
                    const C* xr = x + (long long)n * R + r0 + ln.sub;
#pragma unroll
                    for (int q = 0; q < RPL; ++q) {
                        if (r0 + ln.sub + q * LPE < R) {
                            const C xv = __ldg(xr + q * LPE);
                            acc[q].x = fma(zx, xv.x, acc[q].x); acc[q].x = fma(-zy, xv.y, acc[q].x);
                            acc[q].y = fma(zx, xv.y, acc[q].y); acc[q].y = fma(zy, xv.x, acc[q].y);
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
#pragma unroll
            for (int off = LPE; off < 32; off <<= 1) {
                const C t = shfl_xor2(acc[q], off);
                acc[q].x += t.x; acc[q].y += t.y;
            }
            const int rr = r0 + ln.sub + q * LPE;
            if (ln.grp == 0 && rr < R) y[m * R + rr] = acc[q];
        }
    }
}

// Single right-hand side (GMRES products): warp per row, each lane takes
// entries lane, lane + 32, ... in unrolled groups of 4 (values, columns, then
// the 4 x gathers in flight together); fixed order => deterministic.
template <class C>
__global__ void __launch_bounds__(256) near1_kernel(const int64_t* __restrict__ rowp, const int32_t* __restrict__ col,
                                                    const C* __restrict__ val, const C* __restrict__ x, long long N,
                                                    C* __restrict__ y) {
    const long long m = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / 32;
    if (m >= N) return;
    const int lane = threadIdx.x & 31;
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

// ------------------------------------------ H6 near SpMV, 4-row blocks
// Warp per block of 4 rows (Morton-ordered RWGs); column groups of LPE
// lanes walk the block's union columns, each lane holding RPL right-hand
// sides: one x load feeds the 4 rows (x reuse 4 x fill), the 4 values of a
// column are one contiguous 64 B group (broadcast within the lane group).
// Fixed summation order => deterministic.
#ifndef AIM_NB4_MINB
#define AIM_NB4_MINB 2
#endif
template <int LPE, int RPL, class C>
__global__ void __launch_bounds__(256, AIM_NB4_MINB) near_b4_kernel(const int32_t* __restrict__ rows,
                                                      const int64_t* __restrict__ bptr,
                                                      const int32_t* __restrict__ bcol,
                                                      const C* __restrict__ bval,
                                                      const C* __restrict__ x, long long nblk, int R,
                                                      C* __restrict__ y) {
    using L = Lanes<LPE, RPL>;
    const long long b = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / 32;
    if (b >= nblk) return;
    const L ln;
    const long long e0 = bptr[b], e1 = bptr[b + 1];
    for (int r0 = 0; r0 < R; r0 += L::RC) {
        C acc[4][RPL];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int q = 0; q < RPL; ++q) acc[i][q] = mkc<C>(0, 0);
        // columns staged 32 at a time: lane e loads column e's index and its
        // 4 values (one coalesced 2 KB read per warp), prefetched one batch
        // ahead; values reach the lane groups by shuffles
        int c_n = 0;
        C v_n[4];
        auto fetch = [&](long long e) {
            const int cnt = (int)min(32LL, e1 - e);
            c_n = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) v_n[i] = mkc<C>(0, 0);
            if (ln.lane < cnt) {
                c_n = __ldcs(&bcol[e + ln.lane]);
                const C* vp = bval + 4 * (e + ln.lane);
#pragma unroll
                for (int i = 0; i < 4; ++i) v_n[i] = __ldcs(vp + i);
            }
        };
        if (e0 < e1) fetch(e0);
        for (long long e = e0; e < e1; e += 32) {
            const int cnt = (int)min(32LL, e1 - e);
            const int c_l = c_n;
            C v_l[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) v_l[i] = v_n[i];
            if (e + 32 < e1) fetch(e + 32);
#pragma unroll 2
            for (int t = ln.grp; t < 32; t += L::G) {
                const int c = __shfl_sync(0xffffffffu, c_l, t);
                C v[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) v[i] = shfl_c(v_l[i], t);
                if (t < cnt) {
                    const C* xr = x + (long long)c * R + r0 + ln.sub;
#pragma unroll
                    for (int q = 0; q < RPL; ++q) {
                        if (r0 + ln.sub + q * LPE < R) {
                            const C xv = __ldg(xr + q * LPE);
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                acc[i][q].x = fma(v[i].x, xv.x, acc[i][q].x);
                                acc[i][q].x = fma(-v[i].y, xv.y, acc[i][q].x);
                                acc[i][q].y = fma(v[i].x, xv.y, acc[i][q].y);
                                acc[i][q].y = fma(v[i].y, xv.x, acc[i][q].y);
                            }
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int off = LPE; off < 32; off <<= 1)
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int q = 0; q < RPL; ++q) {
                    const C t = shfl_xor2(acc[i][q], off);
                    acc[i][q].x += t.x;
                    acc[i][q].y += t.y;
                }
        if (ln.grp == 0) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int row = rows[4 * b + i];
#pragma unroll
                for (int q = 0; q < RPL; ++q) {
                    const int rr = r0 + ln.sub + q * LPE;
                    if (row >= 0 && rr < R) y[(long long)row * R + rr] = acc[i][q];
                }
            }
        }
    }
}

// ------------------------------ H6 near SpMM on the FP64 tensor cores
// Warp per block of 8*MT rows (build_near_mma): each chunk of 4 union columns
// is one k-step of mma.m8n8k4.f64 per m-tile, with A = the m-tile's 8x4
// values (lane l holds row l/4, column l%4: bit l of the chunk's mask word,
// packed value popc(mask below l)) and B = x[4 columns][8 RHS] (lane l:
// column l%4, RHS l/4).  C fragment: lane l holds row l/4, RHS 2(l%4) + {0,1}.
// Complex product with three real MMAs per 8-RHS tile (Gauss):
//   T1 = Zr Xr,  T2 = Zi Xi,  T3 = (Zr + Zi)(Xr + Xi);  re = T1 - T2, im = T3 - T1 - T2.
// The masks and columns of a window of 8 chunks are one coalesced load per
// lane (prefetched two windows ahead, handed out by shuffles).
// Fixed order => deterministic.
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(c0), "+d"(c1)
        : "d"(a), "d"(b));
}

// The operands are staged through shared memory by cp.async: every lane owns
// a private ring of D chunk slots (its MT A values and its NT x values per
// chunk), so D chunks per warp are in flight while the MMAs of the oldest
// run, and no register arrays are held across the wait.  Absent values and
// padding columns are zero-filled by plain shared stores.  Chunk j lives in
// slot j % D; after consuming chunk c the lane issues chunk c + D into the
// freed slot, so exactly D - 1 newer copy groups are pending at every wait.
// Blocks of 16 rows (MT = 2) share each x fragment between two m-tiles.
// values stream past L1 (.cg); x rows are re-read by neighbouring blocks of
// the same CTA, so they are cached in L1 (.ca)
__device__ __forceinline__ void cpa16_cg(void* sdst, const void* gsrc) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cpa16_ca(void* sdst, const void* gsrc) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

#ifndef AIM_NM_DEPTH
#define AIM_NM_DEPTH 4
#endif
constexpr int kNmWarps = 4;               // warps per CTA of near_mma_kernel
constexpr int kNmDepth = AIM_NM_DEPTH;    // ring depth (chunks in flight per warp), <= 8
template <int MT, int NT>
constexpr size_t near_mma_smem() { return sizeof(double2) * kNmWarps * kNmDepth * (MT + NT) * 32; }

template <int MT, int NT>
__global__ void __launch_bounds__(32 * kNmWarps) near_mma_kernel(const int32_t* __restrict__ rows,
                                                              const int64_t* __restrict__ cptr,
                                                              const int64_t* __restrict__ vptr,
                                                              const uint32_t* __restrict__ cmask,
                                                              const int32_t* __restrict__ ccol,
                                                              const double2* __restrict__ val,
                                                              const double2* __restrict__ x, long long nblk, int R,
                                                              double2* __restrict__ y) {
    // ring depth D; metadata windows of W = 8 chunks (one column per lane)
    constexpr int D = kNmDepth, W = 8, SL = (MT + NT) * 32;   // SL: slot stride (double2)
    static_assert(D >= 1 && D <= W, "ring depth");
    extern __shared__ __align__(16) double2 nm_sm[];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const long long b = (long long)blockIdx.x * kNmWarps + wid;
    if (b >= nblk) return;
    // this lane's slot u: A of m-tile q at ring[u*SL + q*32], x tile n at ring[u*SL + (MT+n)*32]
    double2* ring = nm_sm + (size_t)wid * D * SL + lane;
    const uint32_t below = (1u << lane) - 1u;
    // 32-bit offsets: nnzN < 2^31 (plan check) and N R < 2^31 (launch check)
    const int c0 = (int)cptr[b], c1 = (int)cptr[b + 1];
    auto meta = [&](int w, int& colw, uint32_t& mw) {
        colw = (4 * w + lane < 4 * c1) ? __ldcs(&ccol[4 * w + lane]) : -1;
        mw = (lane < W * MT && MT * w + lane < MT * c1) ? __ldcs(&cmask[MT * w + lane]) : 0u;
    };
    for (int r0 = 0; r0 < R; r0 += 8 * NT) {
        const double2* xr0 = x + r0 + g;
        int vo = (int)vptr[b];
        // issue the chunk at position j of the window described by (colw, mw) into slot s
        auto issue = [&](int colw, uint32_t mw, int j, int slot) {
            const int col = __shfl_sync(0xffffffffu, colw, 4 * j + t);
            double2* sl = ring + slot * SL;
#pragma unroll
            for (int q = 0; q < MT; ++q) {
                const uint32_t m = __shfl_sync(0xffffffffu, mw, MT * j + q);
                if (m >> lane & 1u) cpa16_cg(sl + q * 32, val + vo + __popc(m & below));
                else sl[q * 32] = make_double2(0.0, 0.0);
                vo += __popc(m);
            }
#pragma unroll
            for (int n = 0; n < NT; ++n) {
                if (col >= 0 && r0 + 8 * n + g < R) cpa16_ca(sl + (MT + n) * 32, xr0 + (col * R + 8 * n));
                else sl[(MT + n) * 32] = make_double2(0.0, 0.0);
            }
            cpa_commit();
        };
        double T1[MT][NT][2], T2[MT][NT][2], T3[MT][NT][2];
#pragma unroll
        for (int q = 0; q < MT; ++q)
#pragma unroll
            for (int n = 0; n < NT; ++n)
#pragma unroll
                for (int i = 0; i < 2; ++i) T1[q][n][i] = T2[q][n][i] = T3[q][n][i] = 0.0;
        int colw, colw_n;
        uint32_t mw, mw_n;
        meta(c0, colw, mw);
        meta(c0 + W, colw_n, mw_n);
#pragma unroll
        for (int u = 0; u < D; ++u) issue(colw, mw, u, u);
        for (int w = c0; w < c1; w += W) {
            int colw_nn;
            uint32_t mw_nn;
            meta(w + 2 * W, colw_nn, mw_nn);
#pragma unroll
            for (int u = 0; u < W; ++u) {
                // chunk w + u sits in slot u % D; chunk w + u + D replaces it
                cpa_wait<D - 1>();
                const double2* sl = ring + (u % D) * SL;
                double2 a[MT], xv[NT];
#pragma unroll
                for (int q = 0; q < MT; ++q) a[q] = sl[q * 32];
#pragma unroll
                for (int n = 0; n < NT; ++n) xv[n] = sl[(MT + n) * 32];
                if (u + D < W) issue(colw, mw, u + D, u % D);   // zero-filled past c1
                else issue(colw_n, mw_n, u + D - W, u % D);
#pragma unroll
                for (int n = 0; n < NT; ++n) {
                    const double xs = xv[n].x + xv[n].y;
#pragma unroll
                    for (int q = 0; q < MT; ++q) {
                        dmma(T1[q][n][0], T1[q][n][1], a[q].x, xv[n].x);
                        dmma(T2[q][n][0], T2[q][n][1], a[q].y, xv[n].y);
                        dmma(T3[q][n][0], T3[q][n][1], a[q].x + a[q].y, xs);
                    }
                }
            }
            colw = colw_n;
            mw = mw_n;
            colw_n = colw_nn;
            mw_n = mw_nn;
        }
        cpa_wait<0>();
#pragma unroll
        for (int q = 0; q < MT; ++q) {
            const int row = rows[8 * MT * b + 8 * q + g];
            if (row < 0) continue;
#pragma unroll
            for (int n = 0; n < NT; ++n)
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const int rr = r0 + 8 * n + 2 * t + i;
                    if (rr < R)
                        y[(long long)row * R + rr] = make_double2(T1[q][n][i] - T2[q][n][i],
                                                                  T3[q][n][i] - T1[q][n][i] - T2[q][n][i]);
                }
        }
    }
}

// ------------------------------ H5 interpolation on the FP64 tensor cores
// y[m, r] += j k eta0 sum_{u, comp} w'[m, u, comp] Phi[comp][g(m, u)][r] (w'_phi =
// -w_phi / k^2) as a block-sparse product (build_interp_mma): warp per block of
// 8*MT RWGs, one chunk per union stencil node, the 4 components are the k
// extent of mma.m8n8k4.f64.  A = real weights (lane l: row l/4, comp l%4, bit l
// of the chunk mask, packed value popc(mask below l)); B = Phi[comp][node][8 RHS]
// (lane l: comp l%4, RHS l/4): real and imaginary parts are two MMAs.  The same
// per-lane cp.async ring as near_mma_kernel; a node index per chunk and MT
// masks, windows of 8 chunks handed out by shuffles.
__device__ __forceinline__ void cpa8_ca(void* sdst, const void* gsrc) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gsrc) : "memory");
}

template <int MT, int NT>
constexpr size_t interp_mma_smem() { return sizeof(double2) * kNmWarps * kNmDepth * (MT + NT) * 32; }

template <int MT, int NT>
__global__ void __launch_bounds__(32 * kNmWarps) interp_mma_kernel(const int32_t* __restrict__ rows,
                                                                const int64_t* __restrict__ cptr,
                                                                const int64_t* __restrict__ vptr,
                                                                const uint32_t* __restrict__ cmask,
                                                                const int32_t* __restrict__ cnode,
                                                                const double* __restrict__ val,
                                                                const double2* __restrict__ Phi, long long Ng,
                                                                long long nblk, int R, double keta,
                                                                double2* __restrict__ y) {
    constexpr int D = kNmDepth, W = 8, SL = (MT + NT) * 32;
    static_assert(D >= 1 && D <= W, "ring depth");
    extern __shared__ __align__(16) double2 nm_sm[];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const long long b = (long long)blockIdx.x * kNmWarps + wid;
    if (b >= nblk) return;
    double2* ring = nm_sm + (size_t)wid * D * SL + lane;
    const uint32_t below = (1u << lane) - 1u;
    const int c0 = (int)cptr[b], c1 = (int)cptr[b + 1];
    auto meta = [&](int w, int& nodew, uint32_t& mw) {
        nodew = (lane < W && w + lane < c1) ? __ldcs(&cnode[w + lane]) : -1;
        mw = (lane < W * MT && MT * w + lane < MT * c1) ? __ldcs(&cmask[MT * w + lane]) : 0u;
    };
    for (int r0 = 0; r0 < R; r0 += 8 * NT) {
        // lane's B column: component t, rhs r0 + 8 n + g
        const double2* ph = Phi + (long long)t * Ng * R + r0 + g;
        int vo = (int)vptr[b];
        auto issue = [&](int nodew, uint32_t mw, int j, int slot) {
            const int node = __shfl_sync(0xffffffffu, nodew, j);
            double2* sl = ring + slot * SL;
#pragma unroll
            for (int q = 0; q < MT; ++q) {
                const uint32_t m = __shfl_sync(0xffffffffu, mw, MT * j + q);
                if (m >> lane & 1u) cpa8_ca(sl + q * 32, val + vo + __popc(m & below));
                else sl[q * 32].x = 0.0;
                vo += __popc(m);
            }
#pragma unroll
            for (int n = 0; n < NT; ++n) {
                if (node >= 0 && r0 + 8 * n + g < R) cpa16_ca(sl + (MT + n) * 32, ph + ((long long)node * R + 8 * n));
                else sl[(MT + n) * 32] = make_double2(0.0, 0.0);
            }
            cpa_commit();
        };
        double Yr[MT][NT][2], Yi[MT][NT][2];
#pragma unroll
        for (int q = 0; q < MT; ++q)
#pragma unroll
            for (int n = 0; n < NT; ++n)
#pragma unroll
                for (int i = 0; i < 2; ++i) Yr[q][n][i] = Yi[q][n][i] = 0.0;
        int nw, nw_n;
        uint32_t mw, mw_n;
        meta(c0, nw, mw);
        meta(c0 + W, nw_n, mw_n);
#pragma unroll
        for (int u = 0; u < D; ++u) issue(nw, mw, u, u);
        for (int w = c0; w < c1; w += W) {
            int nw_nn;
            uint32_t mw_nn;
            meta(w + 2 * W, nw_nn, mw_nn);
#pragma unroll
            for (int u = 0; u < W; ++u) {
                cpa_wait<D - 1>();
                const double2* sl = ring + (u % D) * SL;
                double a[MT];
                double2 xv[NT];
#pragma unroll
                for (int q = 0; q < MT; ++q) a[q] = sl[q * 32].x;
#pragma unroll
                for (int n = 0; n < NT; ++n) xv[n] = sl[(MT + n) * 32];
                if (u + D < W) issue(nw, mw, u + D, u % D);
                else issue(nw_n, mw_n, u + D - W, u % D);
#pragma unroll
                for (int n = 0; n < NT; ++n)
#pragma unroll
                    for (int q = 0; q < MT; ++q) {
                        dmma(Yr[q][n][0], Yr[q][n][1], a[q], xv[n].x);
                        dmma(Yi[q][n][0], Yi[q][n][1], a[q], xv[n].y);
                    }
            }
            nw = nw_n;
            mw = mw_n;
            nw_n = nw_nn;
            mw_n = mw_nn;
        }
        cpa_wait<0>();
#pragma unroll
        for (int q = 0; q < MT; ++q) {
            const int row = rows[8 * MT * b + 8 * q + g];
            if (row < 0) continue;
#pragma unroll
            for (int n = 0; n < NT; ++n)
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const int rr = r0 + 8 * n + 2 * t + i;
                    if (rr < R) {
                        double2* yp = y + (long long)row * R + rr;
                        const double2 o = *yp;   // near rows written before (accumulate)
                        *yp = make_double2(o.x - keta * Yi[q][n][i], o.y + keta * Yr[q][n][i]);
                    }
                }
        }
    }
}

// The tensor-core interpolation is opt-in (AIM_INTERP_KERNEL=mma, complex128,
// R >= 8, accumulating onto the near rows): measured on C2 it is slower than
// the gather kernel (0.253 vs 0.233 ms; chunk fill 0.26 at 16 rows), so the
// gather kernel is the default.
// Single right-hand side, component-interleaved potentials: Phi_i[g][4]
// (one 64-byte record per grid node, written by phi_interleave_kernel).  A
// lane pair shares a stencil node: the even lane loads its x, y potentials
// and weights, the odd lane its z, phi ones, so one warp instruction reads 16
// nodes' complete 64-byte records -- four runs of 256 contiguous bytes
// (4 consecutive z nodes) instead of eight 64-byte runs per component -- and
// the weights of 16 nodes as 512 contiguous bytes.  About 40 L1 wavefronts
// per row instead of about 110 for the component-major gather
// (interp1_kernel); fixed shuffle order => deterministic.
__global__ void __launch_bounds__(256) phi_interleave_kernel(const double2* __restrict__ Phi, long long Ng,
                                                             double2* __restrict__ Pi) {
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= Ng) return;
    double2 v[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) v[c] = __ldcs(&Phi[c * Ng + g]);
    double2* o = Pi + 4 * g;
#pragma unroll
    for (int c = 0; c < 4; ++c) o[c] = v[c];
}

template <int M>
__global__ void __launch_bounds__(256) interp1i_kernel(const double2* __restrict__ Pi, const double* __restrict__ W,
                                                       const int32_t* __restrict__ node0, int Ny, int Nz, long long N,
                                                       double keta, double ik2, int accumulate,
                                                       const int32_t* __restrict__ wrow, double2* __restrict__ y) {
    constexpr int M1 = M + 1, S = M1 * M1 * M1, KI = (S + 15) / 16;   // node rounds of 16
    const long long m = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / 32;
    if (m >= N) return;
    const int lane = threadIdx.x & 31, half = lane & 1, v = lane >> 1;
    const long long g0 = node0[m];
    const long long wr = wrow ? (long long)__ldg(&wrow[m]) : m;
    const double* W2 = W + 4 * wr * S;
    double2 w[KI], f[KI][2];
#pragma unroll
    for (int k = 0; k < KI; ++k) {
        const int u = v + 16 * k;
        double b0 = 0, b1 = 0;
        // volatile: every load of the row is issued before the first FMA
        if (u < S)
            asm volatile("ld.global.cs.v2.f64 {%0, %1}, [%2];\n" : "=d"(b0), "=d"(b1) : "l"(W2 + 4 * u + 2 * half));
        w[k] = make_double2(b0, b1);
    }
#pragma unroll
    for (int k = 0; k < KI; ++k) {
        const int u = v + 16 * k;
        f[k][0] = f[k][1] = make_double2(0, 0);
        if (u < S) {
            const int ui = u / (M1 * M1), uj = (u / M1) % M1, uk = u % M1;
            const double* src = reinterpret_cast<const double*>(Pi + 4 * (g0 + ((long long)ui * Ny + uj) * Nz + uk) + 2 * half);
            double a0, a1, a2, a3;
            asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];\n"
                         : "=d"(a0), "=d"(a1), "=d"(a2), "=d"(a3)
                         : "l"(src));
            f[k][0] = make_double2(a0, a1);
            f[k][1] = make_double2(a2, a3);
        }
    }
    // even lane: w_x Phi_x + w_y Phi_y; odd lane: w_z Phi_z - k^-2 w_phi Phi_phi
    const double s1 = half ? -ik2 : 1.0;
    double2 a = make_double2(0, 0);
#pragma unroll
    for (int k = 0; k < KI; ++k) {
        a.x = fma(w[k].x, f[k][0].x, a.x); a.y = fma(w[k].x, f[k][0].y, a.y);
        a.x = fma(s1 * w[k].y, f[k][1].x, a.x); a.y = fma(s1 * w[k].y, f[k][1].y, a.y);
    }
    double2 tot = make_double2(-keta * a.y, keta * a.x);
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        tot.x += __shfl_xor_sync(0xffffffffu, tot.x, off);
        tot.y += __shfl_xor_sync(0xffffffffu, tot.y, off);
    }
    if (lane == 0) {
        if (accumulate) {
            const double2 o = y[m];
            tot.x += o.x;
            tot.y += o.y;
        }
        y[m] = tot;
    }
}

// Interleaved interpolation (R = 1, complex128, M <= 4): Phi -> Phi_i in the
// scratch buffer, then interp1i_kernel.  AIM_INTERP_IL=0 keeps interp1_kernel.
static bool interp_interleaved(const aim_plan* p, int R) {
    const char* e = getenv("AIM_INTERP_IL");
    if (e && e[0] == '0') return false;
    return R == 1 && p->prec == AIM_C128 && p->M <= 4 && p->W1 != nullptr;
}

static void launch_interp_il(aim_plan* p, const double2* Phi, double2* y, bool accumulate, cudaStream_t s) {
    double2* Pi = p->W1;   // free after the x inverse pass; 4 Px Ny Nz >= 4 Ng elements
    phi_interleave_kernel<<<nblk(p->Ng, 256), 256, 0, s>>>(Phi, p->Ng, Pi);
    note_launch("phi_interleave");
    const double keta = p->k * eta0(), ik2 = 1.0 / (p->k * p->k);
    const int32_t* wrow = p->cp_on ? p->cp_wrow : nullptr;
    const unsigned grid = nblk(p->N * 32, 256);
    switch (p->M) {
#define II(MM) case MM: interp1i_kernel<MM><<<grid, 256, 0, s>>>(Pi, p->W, p->node0, p->dims[1], p->dims[2], p->N, keta, ik2, accumulate ? 1 : 0, wrow, y); break;
        II(1) II(2) II(3) II(4)
#undef II
    }
}

constexpr int kInterpMmaRhs = 8;

template <class C>
static void launch_interp_t(aim_plan* p, const C* Phi, C* y, int R, bool accumulate, cudaStream_t s) {
    if constexpr (sizeof(C) == 16) {
        const char* e = getenv("AIM_INTERP_KERNEL");
        if (R >= kInterpMmaRhs && accumulate && e && !strcmp(e, "mma")) {
            if (p->N * (long long)R >= (1LL << 31) || p->Ng * 4LL * R >= (1LL << 40))
                throw Error(AIM_E_ARG, "interp_mma: index range");
            build_interp_mma(p, s);
            const double keta = p->k * eta0();
#define IM_CALL(MT, NT)                                                                                            \
    {                                                                                                              \
        static unsigned long long attr = 0; /* per device */                                                      \
        if (!(attr >> (p->device & 63) & 1ULL)) {                                                                  \
            AIM_CUDA(cudaFuncSetAttribute(interp_mma_kernel<MT, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,   \
                                          (int)interp_mma_smem<MT, NT>()));                                        \
            attr |= 1ULL << (p->device & 63);                                                                      \
        }                                                                                                          \
        interp_mma_kernel<MT, NT><<<nblk(p->im_count, kNmWarps), 32 * kNmWarps, interp_mma_smem<MT, NT>(), s>>>(   \
            p->im_rows, p->im_cptr, p->im_vptr, p->im_mask, p->im_node, p->im_val, (const double2*)Phi, p->Ng,     \
            p->im_count, R, keta, (double2*)y);                                                                    \
    }
            if (p->im_mt == 1) {
                if (R <= 8) IM_CALL(1, 1)
                else IM_CALL(1, 2)
            } else {
                if (R <= 8) IM_CALL(2, 1)
                else IM_CALL(2, 2)
            }
#undef IM_CALL
            return;
        }
    }
    const unsigned grid = nblk(p->N * 32, 256);
    const double keta = p->k * eta0(), ik2 = 1.0 / (p->k * p->k);
    const Real<C>* W = (const Real<C>*)(sizeof(C) == 16 ? (const void*)p->W : (const void*)p->W32);
    if (R == 1 && p->M <= 4) {
#ifndef AIM_INTERP1_RW
#define AIM_INTERP1_RW 2
#endif
        constexpr int RW = AIM_INTERP1_RW;   // rows per warp
        const unsigned grid1 = nblk((p->N + RW - 1) / RW * 32, 256);
        const int32_t* wrow = p->cp_on ? p->cp_wrow : nullptr;
        switch (p->M) {
#define I1(MM) case MM: interp1_kernel<MM, RW, C><<<grid1, 256, 0, s>>>(Phi, W, p->node0, p->Ng, p->dims[1], p->dims[2], p->N, keta, ik2, accumulate ? 1 : 0, wrow, y); break;
            I1(1) I1(2) I1(3) I1(4)
#undef I1
        }
        return;
    }
#define IN_CALL(LPE, RPL)                                                                                       \
    interp_kernel<MM, LPE, RPL, C><<<grid, 256, 0, s>>>(Phi, W, p->node0, p->Ng, p->dims[1], p->dims[2], p->N, R, \
                                                        keta, ik2, accumulate ? 1 : 0, y)
#define IN_M(MMV)                            \
    if (p->M == MMV) {                       \
        constexpr int MM = MMV;              \
        AIM_LANE_DISPATCH_GATHER(R, IN_CALL) \
        return;                              \
    }
    IN_M(1) IN_M(2) IN_M(3) IN_M(4) IN_M(5) IN_M(6)
#undef IN_M
#undef IN_CALL
    throw Error(AIM_E_ARG, "unsupported M");
}

void launch_interp(aim_plan* p, const void* Phi, void* y, int R, bool accumulate, cudaStream_t s) {
    if (interp_interleaved(p, R)) launch_interp_il(p, (const double2*)Phi, (double2*)y, accumulate, s);
    else if (p->prec == AIM_C64) launch_interp_t(p, (const float2*)Phi, (float2*)y, R, accumulate, s);
    else launch_interp_t(p, (const double2*)Phi, (double2*)y, R, accumulate, s);
    note_launch("interp");
}

// Multi-RHS products use the 4-row blocked layout (x reuse across rows);
// below kNearBlockRhs right-hand sides the plain CSR (fewer value bytes).
constexpr int kNearBlockRhs = 4;

// complex128 products with >= kNearMmaRhs right-hand sides use the FP64
// tensor-core kernel (8-row blocks, packed values).  AIM_NEAR_KERNEL=b4|csr
// in the environment forces another kernel (A/B timing only).
constexpr int kNearMmaRhs = 8;
static int near_override() {
    const char* e = getenv("AIM_NEAR_KERNEL");
    return !e ? 0 : !strcmp(e, "b4") ? 1 : !strcmp(e, "csr") ? 2 : 0;
}

template <class C>
static void launch_near_t(aim_plan* p, const C* x, C* y, int R, cudaStream_t s) {
    const bool c64 = sizeof(C) == 8;
    const int ov = near_override();
    if constexpr (sizeof(C) == 16) {
        if (R >= kNearMmaRhs && ov == 0) {
            build_near_mma(p, s);
            if (p->N * (long long)R >= (1LL << 31)) throw Error(AIM_E_ARG, "near_mma: N * nrhs exceeds 2^31");
#define NM_CALL(MT, NT)                                                                                        \
    {                                                                                                          \
        static unsigned long long attr = 0; /* per device */                                                  \
        if (!(attr >> (p->device & 63) & 1ULL)) {                                                              \
            AIM_CUDA(cudaFuncSetAttribute(near_mma_kernel<MT, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                          (int)near_mma_smem<MT, NT>()));                                      \
            attr |= 1ULL << (p->device & 63);                                                                  \
        }                                                                                                      \
        near_mma_kernel<MT, NT><<<nblk(p->nm_count, kNmWarps), 32 * kNmWarps, near_mma_smem<MT, NT>(), s>>>(   \
            p->nm_rows, p->nm_cptr, p->nm_vptr, p->nm_mask, p->nm_col, p->nm_val, (const double2*)x,           \
            p->nm_count, R, (double2*)y);                                                                      \
    }
            if (p->nm_mt == 1) {
                if (R <= 8) NM_CALL(1, 1)
                else NM_CALL(1, 2)
            } else {
                if (R <= 8) NM_CALL(2, 1)
                else NM_CALL(2, 2)
            }
#undef NM_CALL
            return;
        }
    }
    if (R >= kNearBlockRhs && ov != 2) {
        build_near_blocks(p, s);
        const unsigned grid = nblk(p->nb_count * 32, 256);
        const C* bval = (const C*)(c64 ? (const void*)p->nb_val32 : (const void*)p->nb_val);
#define NB_CALL(LPE, RPL) \
    near_b4_kernel<LPE, RPL, C><<<grid, 256, 0, s>>>(p->nb_rows, p->nb_ptr, p->nb_col, bval, x, p->nb_count, R, y)
        if (R <= 4) { NB_CALL(2, 2); }
        else if (R <= 8) { NB_CALL(4, 2); }
        else { NB_CALL(8, 2); }
#undef NB_CALL
        return;
    }
    const unsigned grid = nblk(p->N * 32, 256);
    const C* val = (const C*)(c64 ? (const void*)p->nval32 : (const void*)p->nval);
    if (R == 1) {
        near1_kernel<C><<<grid, 256, 0, s>>>(p->nrow, p->ncol, val, x, p->N, y);
        return;
    }
#define NK_CALL(LPE, RPL) near_kernel<LPE, RPL, C><<<grid, 256, 0, s>>>(p->nrow, p->ncol, val, x, p->N, R, y)
    AIM_LANE_DISPATCH_NEAR(R, NK_CALL)
#undef NK_CALL
}

void launch_near(aim_plan* p, const void* x, void* y, int R, cudaStream_t s) {
    if (p->cmp_on) {      // repetition-compressed near field (NEXT-3, k_compress.cu)
        launch_near_cmp(p, x, y, R, s);
        return;
    }
    if (p->prec == AIM_C64) launch_near_t(p, (const float2*)x, (float2*)y, R, s);
    else launch_near_t(p, (const double2*)x, (double2*)y, R, s);
    note_launch("near");
}

// ------------------------------------------------------------ plane wave
__global__ void planewave_kernel(const double* __restrict__ qp, const double* __restrict__ qw,
                                 const int32_t* __restrict__ rt, const double* __restrict__ ra,
                                 const double* __restrict__ rp, long long N, double k, double kx, double ky,
                                 double kz, double px, double py, double pz, double2 E0, double2* __restrict__ V) {
    const long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    double2 acc = make_double2(0, 0);
    for (int side = 0; side < 2; ++side) {
        const int t = rt[2 * n + side];
        const double a = ra[2 * n + side];
        const double* p = rp + 6 * n + 3 * side;
        for (int q = 0; q < 7; ++q) {
            const double* r = qp + (7 * t + q) * 3;
            const double lp = a * ((r[0] - p[0]) * px + (r[1] - p[1]) * py + (r[2] - p[2]) * pz);
            double s, c;
            sincos(k * (kx * r[0] + ky * r[1] + kz * r[2]), &s, &c);  // exp(-j k khat.r) = c - j s
            const double f = qw[7 * t + q] * lp;
            acc.x += f * c;
            acc.y -= f * s;
        }
    }
    V[n] = make_double2(E0.x * acc.x - E0.y * acc.y, E0.x * acc.y + E0.y * acc.x);
}

void launch_planewave(const aim_plan* p, const double* khat, const double* pol, double2 E0, double2* V,
                      cudaStream_t s) {
    planewave_kernel<<<nblk(p->N, 256), 256, 0, s>>>(p->tri_qp, p->tri_qw, p->rwg_t, p->rwg_a, p->rwg_p, p->N,
                                                      p->k, khat[0], khat[1], khat[2], pol[0], pol[1], pol[2], E0,
                                                      V);
    note_launch("planewave");
}

// ------------------------------------------------------- H2-H4 convolution
void ensure_workspace(aim_plan* p, int R) {
    if (p->ws_nrhs >= R) return;
    AIM_CUDA(cudaDeviceSynchronize());
    p->release(p->Q);
    p->release(p->W1);
    p->release(p->W2);
    p->W2 = nullptr;
    const long long Nx = p->dims[0], Ny = p->dims[1], Nz = p->dims[2];
    const long long Px = p->pads[0], Py = p->pads[1];
    // complex64 plans use the same buffers at half the size (float2 elements)
    const long long es = p->prec == AIM_C64 ? 1 : 2;   // element size in 8-byte units
    p->Q = (double2*)p->alloc<float2>(es * 4 * Nx * Ny * Nz * R);
    p->W1 = (double2*)p->alloc<float2>(es * 4 * Px * Ny * Nz * R);
    if (p->planar != 1) p->W2 = (double2*)p->alloc<float2>(es * 4 * Px * Py * Nz * R);
    p->ws_nrhs = R;
    for (auto& g : p->graphs) cudaGraphExecDestroy(g.exec);   // they captured the old buffers
    p->graphs.clear();
}

struct Prof {
    aim_plan* p;
    long long base = -1;
    explicit Prof(aim_plan* pp) : p(pp) {
        if (!p || !p->prof) return;
        while (p->ev_pool.size() < p->ev_used + kProfEvents) {
            cudaEvent_t e;
            AIM_CUDA(cudaEventCreate(&e));
            p->ev_pool.push_back(e);
        }
        base = (long long)p->ev_used;
        p->ev_used += kProfEvents;
        p->prof_count++;
    }
    void mark(int slot, cudaStream_t s) {
        if (base >= 0) AIM_CUDA(cudaEventRecord(p->ev_pool[base + slot], s));
    }
};

static void convolve_impl(aim_plan* p, const void* Q, void* Phi, int R, cudaStream_t s, Prof* pr) {
    const long long Nx = p->dims[0], Ny = p->dims[1], Nz = p->dims[2];
    const int Px = p->pads[0], Py = p->pads[1], Pz = p->pads[2];
    FftPass f{};
    f.prec = p->prec;
    const void* spec = p->prec == AIM_C64 ? (const void*)p->spec32 : (const void*)p->spec;
    // x forward, [4][Nx -> Px][Ny Nz R]
    f.in = Q; f.out = p->W1; f.outer = 4; f.Lin = (int)Nx; f.Lout = Px; f.inner = Ny * Nz * R;
    f.mode = 0; f.ax = p->ax[0]; f.TO = f.TI = 0;
    launch_fft_pass(f, s);
    if (pr) pr->mark(2, s);
    if (p->planar == 1) {
        PlanarPass q{};
        q.prec = p->prec;
        q.W = p->W1; q.Px = Px; q.Ny = (int)Ny; q.Nz = (int)Nz; q.R = R; q.PyH = Py / 2 + 1; q.ay = p->ax[1];
        q.off = 0; q.Pfold = Px;
        q.spec = spec;
        launch_planar_yz(q, s);
    } else {
        // mode 2, one RHS, a compiled plan: the fused y/z pass in place on W1
        if (p->planar == 2 && launch_ymode2(p->W1, p->prec, Px, (int)Ny, (int)Nz, Py, R, spec, p->ax[1], s)) {
            if (pr) pr->mark(3, s);
            f.in = p->W1; f.out = Phi; f.outer = 4; f.Lin = Px; f.Lout = (int)Nx; f.inner = Ny * Nz * R;
            f.mode = 1; f.ax = p->ax[0]; f.TO = f.TI = 0;
            launch_fft_pass(f, s);
            if (pr) pr->mark(4, s);
            return;
        }
        // y forward, [4 Px][Ny -> Py][Nz R]
        f.in = p->W1; f.out = p->W2; f.outer = 4LL * Px; f.Lin = (int)Ny; f.Lout = Py; f.inner = Nz * R;
        f.mode = 0; f.ax = p->ax[1]; f.TO = f.TI = 0;
        launch_fft_pass(f, s);
        if (p->planar == 2) {
            // z convolution as a direct Toeplitz product with G2(kx, ky, |dz|), in place
            launch_ztoeplitz(p->W2, p->prec, Px, Py, (int)Nz, R, 1, 0, Px, Py, spec, s);
        } else {
            // z turnaround in place, [4 Px Py][Nz -> Pz -> Nz][R]
            f.in = p->W2; f.out = p->W2; f.outer = 4LL * Px * Py; f.Lin = (int)Nz; f.Lout = (int)Nz; f.inner = R;
            f.mode = 2; f.ax = p->ax[2]; f.TO = f.TI = 0;
            f.spec = spec; f.Px = Px; f.Py = Py; f.PyH = Py / 2 + 1; f.PzH = Pz / 2 + 1;
            launch_fft_pass(f, s);
        }
        // y inverse, [4 Px][Py -> Ny][Nz R]
        f.in = p->W2; f.out = p->W1; f.outer = 4LL * Px; f.Lin = Py; f.Lout = (int)Ny; f.inner = Nz * R;
        f.mode = 1; f.ax = p->ax[1]; f.TO = f.TI = 0;
        launch_fft_pass(f, s);
    }
    if (pr) pr->mark(3, s);
    // x inverse, [4][Px -> Nx][Ny Nz R]
    f.in = p->W1; f.out = Phi; f.outer = 4; f.Lin = Px; f.Lout = (int)Nx; f.inner = Ny * Nz * R;
    f.mode = 1; f.ax = p->ax[0]; f.TO = f.TI = 0;
    launch_fft_pass(f, s);
    if (pr) pr->mark(4, s);
}

void convolve(aim_plan* p, const void* Q, void* Phi, int R, cudaStream_t s) {
    convolve_impl(p, Q, Phi, R, s, nullptr);
}

// y = Z_eq x.  All stages run in order on the caller's stream: the near-field
// SpMV first (it writes y), then projection, the FFT passes and the
// interpolation, which accumulates the far field into y.  (Running the SpMV
// on a side stream bought nothing: its 14k CTAs occupy every SM and the
// persistent FFT CTAs queue behind them.)
static void matvec_body(aim_plan* p, const void* x, void* y, int R, cudaStream_t s) {
    Prof pr(p);
    pr.mark(0, s);
    // Repetition-compressed single-RHS products: the near field (a sparse x
    // dense product over L2-resident dictionary blocks, not HBM-bound) runs on
    // the side stream beside the projection and the FFT passes (shared-memory /
    // FP64 bound) and joins before the interpolation accumulates into y.
    // AIM_CMP_SIDE=0 runs it in order (A/B); profiled products (aim_profile,
    // per-stage events) run in order so the stage times stay separable.
    const char* es = getenv("AIM_CMP_SIDE");
    if (p->cmp_on && R == 1 && !p->prof && !(es && es[0] == '0')) {
        AIM_CUDA(cudaEventRecord(p->ev_x, s));
        AIM_CUDA(cudaStreamWaitEvent(p->side, p->ev_x, 0));
        pr.mark(7, s);
        launch_near(p, x, y, R, p->side);
        AIM_CUDA(cudaEventRecord(p->ev_n, p->side));
        pr.mark(8, s);
        launch_project(p, x, p->Q, R, s);
        pr.mark(1, s);
        convolve_impl(p, p->Q, p->Q, R, s, &pr);
        pr.mark(5, s);
        AIM_CUDA(cudaStreamWaitEvent(s, p->ev_n, 0));
        launch_interp(p, p->Q, y, R, true, s);
        pr.mark(6, s);
        return;
    }
    // AIM_NEAR_OVL=1 (measured slower, kept opt-in): the near SpMV streams its
    // matrix through shared memory beside the FFT passes (k_near_stream.cu):
    // CTAs on the side stream from the end of the projection take a share of
    // the row chunks, the rest is taken at full occupancy on s after the FFT;
    // both join before the interpolation accumulates into y.
    if (!p->cmp_on && R == 1 && !p->prof && near_overlap_mode() && near_stream_ready(p, s)) {
        near_stream_reset(p, s);
        launch_project(p, x, p->Q, R, s);
        const int a = near_overlap_ctas_per_sm();   // 0: no side launch (A/B of the streamed kernel alone)
        if (a > 0) {
            AIM_CUDA(cudaEventRecord(p->ev_x, s));
            AIM_CUDA(cudaStreamWaitEvent(p->side, p->ev_x, 0));
            launch_near_stream(p, x, y, a, p->side);
            AIM_CUDA(cudaEventRecord(p->ev_n, p->side));
        }
        convolve_impl(p, p->Q, p->Q, R, s, &pr);
        launch_near_stream(p, x, y, 0, s);
        if (a > 0) AIM_CUDA(cudaStreamWaitEvent(s, p->ev_n, 0));
        launch_interp(p, p->Q, y, R, true, s);
        return;
    }
    // AIM_NEAR_PRIO=1: the FFT passes on a high-priority stream, near1 in
    // 128-thread CTAs on the side stream from the end of the projection, so
    // the block scheduler places the persistent FFT CTAs first and fills the
    // rest of every SM with near rows; both join before the interpolation.
    if (!p->cmp_on && R == 1 && !p->prof && near_prio_mode() && p->prec == AIM_C128) {
        if (!p->hi) {
            int lo = 0, hi = 0;
            AIM_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            AIM_CUDA(cudaStreamCreateWithPriority(&p->hi, cudaStreamNonBlocking, hi));
            AIM_CUDA(cudaEventCreateWithFlags(&p->ev_h, cudaEventDisableTiming));
            static unsigned long long attr = 0;  // per device
            const char* en = getenv("AIM_NEAR1_CARVE");   // A/B: 0 = near1 keeps its default carveout
            if (!(attr >> (p->device & 63) & 1ULL) && !(en && en[0] == '0')) {
                AIM_CUDA(cudaFuncSetAttribute(near1_kernel<double2>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
                attr |= 1ULL << (p->device & 63);
            }
        }
        launch_project(p, x, p->Q, R, s);
        AIM_CUDA(cudaEventRecord(p->ev_x, s));
        AIM_CUDA(cudaStreamWaitEvent(p->side, p->ev_x, 0));
        AIM_CUDA(cudaStreamWaitEvent(p->hi, p->ev_x, 0));
        const char* et = getenv("AIM_NEAR_PRIO_T");
        const int nt = et ? atoi(et) : 128;
        near1_kernel<double2><<<nblk(p->N * 32, nt), nt, 0, p->side>>>(p->nrow, p->ncol, p->nval, (const double2*)x,
                                                                       p->N, (double2*)y);
        note_launch("near");
        AIM_CUDA(cudaEventRecord(p->ev_n, p->side));
        convolve_impl(p, p->Q, p->Q, R, p->hi, &pr);
        AIM_CUDA(cudaEventRecord(p->ev_h, p->hi));
        AIM_CUDA(cudaStreamWaitEvent(s, p->ev_h, 0));
        AIM_CUDA(cudaStreamWaitEvent(s, p->ev_n, 0));
        launch_interp(p, p->Q, y, R, true, s);
        return;
    }
    pr.mark(7, s);
    launch_near(p, x, y, R, s);
    pr.mark(8, s);
    launch_project(p, x, p->Q, R, s);
    pr.mark(1, s);
    convolve_impl(p, p->Q, p->Q, R, s, &pr);
    pr.mark(5, s);
    launch_interp(p, p->Q, y, R, true, s);
    pr.mark(6, s);
}

// The product as a CUDA graph (small products are launch
// bound): the first product for an nrhs runs eagerly (it builds lazily
// created tables and sets kernel attributes); later products are captured
// once per (x, y, nrhs) on the plan's stream, instantiated, and replayed with
// an event fork/join onto the caller's stream.  Profiling (aim_profile) and
// AIM_GRAPH=0 run eagerly.
void matvec(aim_plan* p, const void* x, void* y, int R, cudaStream_t s) {
    ensure_workspace(p, R);
    const char* env = getenv("AIM_GRAPH");
    const bool graphs = !(env && env[0] == '0');
    const bool warm = R < (int)p->mv_warm.size() && p->mv_warm[R];
    if (!graphs || p->prof || !warm) {
        matvec_body(p, x, y, R, s);
        if (R >= (int)p->mv_warm.size()) p->mv_warm.resize(R + 1, 0);
        p->mv_warm[R] = 1;
        return;
    }
    aim_plan::MvGraph* g = nullptr;
    for (auto& q : p->graphs)
        if (q.x == x && q.y == y && q.R == R) g = &q;
    if (!g) {
        if (p->graphs.size() >= 128) {
            cudaGraphExecDestroy(p->graphs.front().exec);
            p->graphs.erase(p->graphs.begin());
        }
        cudaGraph_t graph;
        const long long before = launch_counter();
        AIM_CUDA(cudaStreamBeginCapture(p->stream, cudaStreamCaptureModeThreadLocal));
        try {
            matvec_body(p, x, y, R, p->stream);
        } catch (...) {
            cudaStreamEndCapture(p->stream, &graph);
            if (graph) cudaGraphDestroy(graph);
            throw;
        }
        AIM_CUDA(cudaStreamEndCapture(p->stream, &graph));
        cudaGraphExec_t exec;
        const cudaError_t e =
            cudaGraphInstantiate(&exec, graph, near_prio_mode() ? cudaGraphInstantiateFlagUseNodePriority : 0);
        cudaGraphDestroy(graph);
        AIM_CUDA(e);
        const long long nk = launch_counter() - before;
        add_launches(-nk);      // counted when the graph is launched
        p->graphs.push_back({x, y, R, exec, nk});
        g = &p->graphs.back();
    }
    if (!p->gx_fork) {
        AIM_CUDA(cudaEventCreateWithFlags(&p->gx_fork, cudaEventDisableTiming));
        AIM_CUDA(cudaEventCreateWithFlags(&p->gx_join, cudaEventDisableTiming));
    }
    AIM_CUDA(cudaEventRecord(p->gx_fork, s));
    AIM_CUDA(cudaStreamWaitEvent(p->stream, p->gx_fork, 0));
    AIM_CUDA(cudaGraphLaunch(g->exec, p->stream));
    AIM_CUDA(cudaEventRecord(p->gx_join, p->stream));
    AIM_CUDA(cudaStreamWaitEvent(s, p->gx_join, 0));
    add_launches(g->kernels);
}

}  // namespace aim
