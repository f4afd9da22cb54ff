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

#include "aim_internal.cuh"

namespace aim {

static inline unsigned nblk(long long n, int t) { return (unsigned)((n + t - 1) / t); }

__device__ __forceinline__ double2 shfl_xor2(double2 v, int m) {
    return make_double2(__shfl_xor_sync(0xffffffffu, v.x, m), __shfl_xor_sync(0xffffffffu, v.y, m));
}

// ------------------------------------------------------------ H1 projection
// Warp per grid node.  Entries are consumed in batches of 32: every lane first
// loads one entry's index and weights (coalesced / independent), then the
// rhs lanes gather x for the batch (broadcast by shuffles), so each warp keeps
// many independent loads in flight.
template <int M, int RC>
__global__ void __launch_bounds__(256) project_kernel(const int32_t* __restrict__ prow,
                                                      const int32_t* __restrict__ pent,
                                                      const double* __restrict__ W, const double2* __restrict__ x,
                                                      long long Ng, int R, double2* __restrict__ Q) {
    constexpr int S = (M + 1) * (M + 1) * (M + 1);
    constexpr int G = 32 / RC;
    const long long g = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / 32;
    if (g >= Ng) return;
    const int lane = threadIdx.x & 31;
    const int grp = lane / RC, r = lane % RC;
    const int e0 = prow[g], e1 = prow[g + 1];
    const double2* W2 = reinterpret_cast<const double2*>(W);
    for (int r0 = 0; r0 < R; r0 += RC) {
        const int rr = r0 + r;
        const bool act = rr < R;
        double2 a0 = make_double2(0, 0), a1 = a0, a2 = a0, a3 = a0;
        for (int b = e0; b < e1; b += 32) {
            const int cnt = min(32, e1 - b);
            int n_l = 0;
            double2 w01 = make_double2(0, 0), w23 = w01;
            if (lane < cnt) {
                const int ent = __ldg(&pent[b + lane]);
                n_l = ent / S;
                w01 = __ldcs(W2 + 2 * (long long)ent);
                w23 = __ldcs(W2 + 2 * (long long)ent + 1);
            }
            if (RC == 1) {
                if (lane < cnt) {
                    const double2 xv = __ldg(&x[(long long)n_l * R + rr]);
                    a0.x = fma(w01.x, xv.x, a0.x); a0.y = fma(w01.x, xv.y, a0.y);
                    a1.x = fma(w01.y, xv.x, a1.x); a1.y = fma(w01.y, xv.y, a1.y);
                    a2.x = fma(w23.x, xv.x, a2.x); a2.y = fma(w23.x, xv.y, a2.y);
                    a3.x = fma(w23.y, xv.x, a3.x); a3.y = fma(w23.y, xv.y, a3.y);
                }
            } else {
#pragma unroll 4
                for (int t = grp; t < 32; t += G) {
                    const int n = __shfl_sync(0xffffffffu, n_l, t);
                    const double wx = __shfl_sync(0xffffffffu, w01.x, t), wy = __shfl_sync(0xffffffffu, w01.y, t);
                    const double wz = __shfl_sync(0xffffffffu, w23.x, t), wp = __shfl_sync(0xffffffffu, w23.y, t);
                    if (t < cnt && act) {
                        const double2 xv = __ldg(&x[(long long)n * R + rr]);
                        a0.x = fma(wx, xv.x, a0.x); a0.y = fma(wx, xv.y, a0.y);
                        a1.x = fma(wy, xv.x, a1.x); a1.y = fma(wy, xv.y, a1.y);
                        a2.x = fma(wz, xv.x, a2.x); a2.y = fma(wz, xv.y, a2.y);
                        a3.x = fma(wp, xv.x, a3.x); a3.y = fma(wp, xv.y, a3.y);
                    }
                }
            }
        }
#pragma unroll
        for (int off = RC; off < 32; off <<= 1) {
            double2 t;
            t = shfl_xor2(a0, off); a0.x += t.x; a0.y += t.y;
            t = shfl_xor2(a1, off); a1.x += t.x; a1.y += t.y;
            t = shfl_xor2(a2, off); a2.x += t.x; a2.y += t.y;
            t = shfl_xor2(a3, off); a3.x += t.x; a3.y += t.y;
        }
        if (RC == 1) {
            if (lane < 4) {
                const double2 v = lane == 0 ? a0 : lane == 1 ? a1 : lane == 2 ? a2 : a3;
                __stcs(&Q[((long long)lane * Ng + g) * R + rr], v);
            }
        } else if (grp == 0 && act) {
            __stcs(&Q[(0 * Ng + g) * R + rr], a0);
            __stcs(&Q[(1 * Ng + g) * R + rr], a1);
            __stcs(&Q[(2 * Ng + g) * R + rr], a2);
            __stcs(&Q[(3 * Ng + g) * R + rr], a3);
        }
    }
}

static int rhs_chunk(int R) {
    int rc = 1;
    while (rc < R && rc < 32) rc <<= 1;
    return rc;
}

void launch_project(const aim_plan* p, const double2* x, double2* Q, int R, cudaStream_t s) {
    const int rc = rhs_chunk(R);
    const unsigned grid = nblk(p->Ng * 32, 256);
#define PJ(MM, RR) \
    if (p->M == MM && rc == RR) { project_kernel<MM, RR><<<grid, 256, 0, s>>>(p->prow, p->pent, p->W, x, p->Ng, R, Q); note_launch("project"); return; }
#define PJM(MM) PJ(MM, 1) PJ(MM, 2) PJ(MM, 4) PJ(MM, 8) PJ(MM, 16) PJ(MM, 32)
    PJM(1) PJM(2) PJM(3) PJM(4) PJM(5) PJM(6)
#undef PJM
#undef PJ
    throw Error(AIM_E_ARG, "unsupported M");
}

// ------------------------------------------------------ H5 interpolation
// y[m,r] (+)= j k eta0 [sum_xyz sum_u w_{m,u} Phi[u,r] - k^-2 sum_u w^phi_{m,u} Phi^phi[u,r]]
// Warp per RWG row: lane u first loads w_{m,u} (contiguous), then the rhs
// lanes gather the stencil's potentials (weights broadcast by shuffles).
template <int M, int RC>
__global__ void __launch_bounds__(256) interp_kernel(const double2* __restrict__ Phi, const double* __restrict__ W,
                                                     const int32_t* __restrict__ node0, long long Ng, int Ny, int Nz,
                                                     long long N, int R, double keta, double ik2, int accumulate,
                                                     double2* __restrict__ y) {
    constexpr int M1 = M + 1, S = M1 * M1 * M1;
    constexpr int G = 32 / RC;
    const long long m = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / 32;
    if (m >= N) return;
    const int lane = threadIdx.x & 31;
    const int grp = lane / RC, r = lane % RC;
    const long long g0 = node0[m];
    const double2* W2 = reinterpret_cast<const double2*>(W) + 2 * m * S;
    for (int r0 = 0; r0 < R; r0 += RC) {
        const int rr = r0 + r;
        const bool act = rr < R;
        double2 aA = make_double2(0, 0), aP = aA;
        for (int ub = 0; ub < S; ub += 32) {
            const int u_l = ub + lane;
            double2 w01 = make_double2(0, 0), w23 = w01;
            int g_l = 0;
            if (u_l < S) {
                w01 = __ldcs(W2 + 2 * u_l);
                w23 = __ldcs(W2 + 2 * u_l + 1);
                const int ui = u_l / (M1 * M1), uj = (u_l / M1) % M1, uk = u_l % M1;
                g_l = (int)(g0 + ((long long)ui * Ny + uj) * Nz + uk);
            }
            if (RC == 1) {
                if (u_l < S) {
                    const double2 f0 = __ldg(&Phi[(0 * Ng + g_l) * R + rr]);
                    const double2 f1 = __ldg(&Phi[(1 * Ng + g_l) * R + rr]);
                    const double2 f2 = __ldg(&Phi[(2 * Ng + g_l) * R + rr]);
                    const double2 f3 = __ldg(&Phi[(3 * Ng + g_l) * R + rr]);
                    aA.x = fma(w01.x, f0.x, aA.x); aA.y = fma(w01.x, f0.y, aA.y);
                    aA.x = fma(w01.y, f1.x, aA.x); aA.y = fma(w01.y, f1.y, aA.y);
                    aA.x = fma(w23.x, f2.x, aA.x); aA.y = fma(w23.x, f2.y, aA.y);
                    aP.x = fma(w23.y, f3.x, aP.x); aP.y = fma(w23.y, f3.y, aP.y);
                }
            } else {
                const int cnt = min(32, S - ub);
#pragma unroll 4
                for (int t = grp; t < 32; t += G) {
                    const long long g = __shfl_sync(0xffffffffu, g_l, t);
                    const double wx = __shfl_sync(0xffffffffu, w01.x, t), wy = __shfl_sync(0xffffffffu, w01.y, t);
                    const double wz = __shfl_sync(0xffffffffu, w23.x, t), wp = __shfl_sync(0xffffffffu, w23.y, t);
                    if (t < cnt && act) {
                        const double2 f0 = __ldg(&Phi[(0 * Ng + g) * R + rr]);
                        const double2 f1 = __ldg(&Phi[(1 * Ng + g) * R + rr]);
                        const double2 f2 = __ldg(&Phi[(2 * Ng + g) * R + rr]);
                        const double2 f3 = __ldg(&Phi[(3 * Ng + g) * R + rr]);
                        aA.x = fma(wx, f0.x, aA.x); aA.y = fma(wx, f0.y, aA.y);
                        aA.x = fma(wy, f1.x, aA.x); aA.y = fma(wy, f1.y, aA.y);
                        aA.x = fma(wz, f2.x, aA.x); aA.y = fma(wz, f2.y, aA.y);
                        aP.x = fma(wp, f3.x, aP.x); aP.y = fma(wp, f3.y, aP.y);
                    }
                }
            }
        }
        // far = j k eta0 (aA - aP / k^2)
        const double2 f = make_double2(aA.x - aP.x * ik2, aA.y - aP.y * ik2);
        double2 tot = make_double2(-keta * f.y, keta * f.x);
#pragma unroll
        for (int off = RC; off < 32; off <<= 1) {
            const double2 t = shfl_xor2(tot, off);
            tot.x += t.x; tot.y += t.y;
        }
        if (grp == 0 && act) {
            if (accumulate) {
                const double2 o = y[m * R + rr];
                tot.x += o.x; tot.y += o.y;
            }
            y[m * R + rr] = tot;
        }
    }
}

// ------------------------------------------------------- H6 near SpMV
// y[m,r] = sum_{n in near(m)} Z_corr[m,n] x[n,r]; warp per row.  Batches of
// 32 entries: lane e loads (Z, col) of entry e (coalesced, streamed past L1),
// then the rhs lanes gather x (entry broadcast by shuffles); fixed-order
// shuffle reduction at the end.
template <int RC>
__global__ void __launch_bounds__(256) near_kernel(const int64_t* __restrict__ rowp, const int32_t* __restrict__ col,
                                                   const double2* __restrict__ val, const double2* __restrict__ x,
                                                   long long N, int R, double2* __restrict__ y) {
    constexpr int G = 32 / RC;
    const long long m = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / 32;
    if (m >= N) return;
    const int lane = threadIdx.x & 31;
    const int grp = lane / RC, r = lane % RC;
    const long long e0 = rowp[m], e1 = rowp[m + 1];
    for (int r0 = 0; r0 < R; r0 += RC) {
        const int rr = r0 + r;
        const bool act = rr < R;
        double2 aN = make_double2(0, 0);
        for (long long b = e0; b < e1; b += 32) {
            const int cnt = (int)min(32LL, e1 - b);
            double2 z_l = make_double2(0, 0);
            int n_l = 0;
            if (lane < cnt) {
                z_l = __ldcs(&val[b + lane]);
                n_l = __ldcs(&col[b + lane]);
            }
            if (RC == 1) {
                if (lane < cnt) {
                    const double2 xv = __ldg(&x[(long long)n_l * R + rr]);
                    aN.x = fma(z_l.x, xv.x, aN.x); aN.x = fma(-z_l.y, xv.y, aN.x);
                    aN.y = fma(z_l.x, xv.y, aN.y); aN.y = fma(z_l.y, xv.x, aN.y);
                }
            } else {
#pragma unroll 8
                for (int t = grp; t < 32; t += G) {
                    const int n = __shfl_sync(0xffffffffu, n_l, t);
                    const double zx = __shfl_sync(0xffffffffu, z_l.x, t), zy = __shfl_sync(0xffffffffu, z_l.y, t);
                    if (t < cnt && act) {
                        const double2 xv = __ldg(&x[(long long)n * R + rr]);
                        aN.x = fma(zx, xv.x, aN.x); aN.x = fma(-zy, xv.y, aN.x);
                        aN.y = fma(zx, xv.y, aN.y); aN.y = fma(zy, xv.x, aN.y);
                    }
                }
            }
        }
#pragma unroll
        for (int off = RC; off < 32; off <<= 1) {
            const double2 t = shfl_xor2(aN, off);
            aN.x += t.x; aN.y += t.y;
        }
        if (grp == 0 && act) y[m * R + rr] = aN;
    }
}

void launch_interp(const aim_plan* p, const double2* Phi, double2* y, int R, bool accumulate, cudaStream_t s) {
    const int rc = rhs_chunk(R);
    const unsigned grid = nblk(p->N * 32, 256);
    const double keta = p->k * eta0(), ik2 = 1.0 / (p->k * p->k);
#define IN(MM, RR)                                                                                        \
    if (p->M == MM && rc == RR) {                                                                         \
        interp_kernel<MM, RR><<<grid, 256, 0, s>>>(Phi, p->W, p->node0, p->Ng, p->dims[1], p->dims[2], p->N, R, \
                                                   keta, ik2, accumulate ? 1 : 0, y);                     \
        note_launch("interp");                                                                            \
        return;                                                                                           \
    }
#define INM(MM) IN(MM, 1) IN(MM, 2) IN(MM, 4) IN(MM, 8) IN(MM, 16) IN(MM, 32)
    INM(1) INM(2) INM(3) INM(4) INM(5) INM(6)
#undef INM
#undef IN
    throw Error(AIM_E_ARG, "unsupported M");
}

void launch_near(const aim_plan* p, const double2* x, double2* y, int R, cudaStream_t s) {
    const int rc = rhs_chunk(R);
    const unsigned grid = nblk(p->N * 32, 256);
    switch (rc) {
#define NK(RR) case RR: near_kernel<RR><<<grid, 256, 0, s>>>(p->nrow, p->ncol, p->nval, x, p->N, R, y); break;
        NK(1) NK(2) NK(4) NK(8) NK(16) NK(32)
#undef NK
    }
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
    p->Q = p->alloc<double2>(4 * Nx * Ny * Nz * R);
    p->W1 = p->alloc<double2>(4 * Px * Ny * Nz * R);
    if (!p->planar) p->W2 = p->alloc<double2>(4 * Px * Py * Nz * R);
    p->ws_nrhs = R;
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

static void convolve_impl(aim_plan* p, const double2* Q, double2* Phi, int R, cudaStream_t s, Prof* pr) {
    const long long Nx = p->dims[0], Ny = p->dims[1], Nz = p->dims[2];
    const int Px = p->pads[0], Py = p->pads[1], Pz = p->pads[2];
    FftPass f{};
    // x forward, [4][Nx -> Px][Ny Nz R]
    f.in = Q; f.out = p->W1; f.outer = 4; f.Lin = (int)Nx; f.Lout = Px; f.inner = Ny * Nz * R;
    f.mode = 0; f.ax = p->ax[0]; f.TO = f.TI = 0;
    launch_fft_pass(f, s);
    if (pr) pr->mark(2, s);
    if (p->planar) {
        PlanarPass q{};
        q.W = p->W1; q.Px = Px; q.Ny = (int)Ny; q.Nz = (int)Nz; q.R = R; q.PyH = Py / 2 + 1; q.ay = p->ax[1];
        q.spec = p->spec;
        launch_planar_yz(q, s);
    } else {
        // y forward, [4 Px][Ny -> Py][Nz R]
        f.in = p->W1; f.out = p->W2; f.outer = 4LL * Px; f.Lin = (int)Ny; f.Lout = Py; f.inner = Nz * R;
        f.mode = 0; f.ax = p->ax[1]; f.TO = f.TI = 0;
        launch_fft_pass(f, s);
        // z turnaround in place, [4 Px Py][Nz -> Pz -> Nz][R]
        f.in = p->W2; f.out = p->W2; f.outer = 4LL * Px * Py; f.Lin = (int)Nz; f.Lout = (int)Nz; f.inner = R;
        f.mode = 2; f.ax = p->ax[2]; f.TO = f.TI = 0;
        f.spec = p->spec; f.Px = Px; f.Py = Py; f.PyH = Py / 2 + 1; f.PzH = Pz / 2 + 1;
        launch_fft_pass(f, s);
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

void convolve(aim_plan* p, const double2* Q, double2* Phi, int R, cudaStream_t s) {
    convolve_impl(p, Q, Phi, R, s, nullptr);
}

// y = Z_eq x.  The near-field SpMV (memory bound) runs on the plan's side
// stream concurrently with the projection + FFT passes (FP64-ALU heavy);
// the interpolation adds the far field to its result.
void matvec(aim_plan* p, const double2* x, double2* y, int R, cudaStream_t s) {
    ensure_workspace(p, R);
    Prof pr(p);
    pr.mark(0, s);
    AIM_CUDA(cudaEventRecord(p->ev_x, s));
    AIM_CUDA(cudaStreamWaitEvent(p->side, p->ev_x, 0));
    pr.mark(7, p->side);
    launch_near(p, x, y, R, p->side);
    pr.mark(8, p->side);
    AIM_CUDA(cudaEventRecord(p->ev_n, p->side));
    launch_project(p, x, p->Q, R, s);
    pr.mark(1, s);
    convolve_impl(p, p->Q, p->Q, R, s, &pr);
    AIM_CUDA(cudaStreamWaitEvent(s, p->ev_n, 0));
    pr.mark(5, s);
    launch_interp(p, p->Q, y, R, true, s);
    pr.mark(6, s);
}

}  // namespace aim
