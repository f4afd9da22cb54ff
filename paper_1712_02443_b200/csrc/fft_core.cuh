// Shared-memory mixed-radix Stockham FFT core used by the FFT pass kernels
// (step (ii) of the AIM matvec, eq. AIM_step2).
//
// NL independent lines of length P live in shared memory laid out [P][NL]
// (line index fastest => conflict-free butterflies), ping-ponged between two
// buffers; each stage applies twiddles + the radix-R DFT in registers and
// stores in Stockham (self-sorting) order.
//   stage: j in [0, P/R), k = j mod Ns
//     a_t = x[j + t P/R] * w^{t k P/(Ns R)},  b = DFT_R(a),
//     y[(j div Ns) Ns R + k + u Ns] = b_u
#pragma once

#include <cuda_runtime.h>

#include "aim_internal.cuh"
#include "cplx.cuh"

namespace aim {
#ifdef AIM_BOUNDS_DEBUG
__device__ int g_aim_dbg = 0;
#endif

// cos / sin (2 pi (m+1) / R), m = 0 .. (R-3)/2, for the odd radices
template <int R>
__device__ __forceinline__ constexpr double oc(int m) {
    return R == 3 ? -0.5
         : R == 5 ? (m == 0 ? 0.309016994374947451263 : -0.809016994374947451263)
                  : (m == 0 ? 0.623489801858733483364 : m == 1 ? -0.222520933956314392876 : -0.900968867902419145999);
}
template <int R>
__device__ __forceinline__ constexpr double os(int m) {
    return R == 3 ? 0.866025403784438596588
         : R == 5 ? (m == 0 ? 0.951056516295153531182 : 0.587785252292473137103)
                  : (m == 0 ? 0.781831482468029803634 : m == 1 ? 0.974927912181823619342 : 0.433883739117558120402);
}

// Twiddles of the composite in-register radices: c_rtw[rtw_off(R) + j] =
// exp(-2 pi i j / R) (filled once per device by init_radix_twiddles()).
constexpr int kRtwTotal = 6 + 8 + 9 + 10 + 12 + 14 + 15 + 16 + 28;
__host__ __device__ constexpr int rtw_off(int R) {
    return R == 6 ? 0 : R == 8 ? 6 : R == 9 ? 14 : R == 10 ? 23 : R == 12 ? 33 : R == 14 ? 45 : R == 15 ? 59
         : R == 16 ? 74 : 90;
}
__constant__ double2 c_rtw[kRtwTotal];

// composite R = A * B, A the first (prime-power) factor
template <int R>
struct Split {
    static constexpr int A = R == 16 ? 4 : R == 12 ? 4 : R == 28 ? 4 : R == 8 ? 2 : (R % 2 == 0) ? 2 : 3;
    static constexpr int B = R / A;
};

// b_u = sum_t a_t exp(sign 2 pi i t u / R), in place
template <int R, class C>
__device__ __forceinline__ void dft(C* a, double sign_d) {
    using T = Real<C>;
    const T sign = (T)sign_d;
    if constexpr (R == 1) {
    } else if constexpr (R != 2 && R != 3 && R != 4 && R != 5 && R != 7) {
        // decimation in time inside registers: Y_r = DFT_B(a[A m + r]),
        // X[k + B s] = DFT_A over r of W_R^{r k} Y_r[k]
        constexpr int A = Split<R>::A, B = Split<R>::B;
        C y[A][B];
#pragma unroll
        for (int r = 0; r < A; ++r) {
#pragma unroll
            for (int m = 0; m < B; ++m) y[r][m] = a[A * m + r];
            dft<B>(y[r], sign_d);
        }
#pragma unroll
        for (int k = 0; k < B; ++k) {
            C t[A];
#pragma unroll
            for (int r = 0; r < A; ++r) {
                t[r] = y[r][k];
                if ((r * k) % R) {
                    C w = cvt<C>(c_rtw[rtw_off(R) + (r * k) % R]);
                    if (sign > 0) w.y = -w.y;
                    t[r] = cmul(t[r], w);
                }
            }
            dft<A>(t, sign_d);
#pragma unroll
            for (int q = 0; q < A; ++q) a[k + B * q] = t[q];
        }
    } else if constexpr (R == 2) {
        const C t = a[0];
        a[0] = cadd(t, a[1]);
        a[1] = csub(t, a[1]);
    } else if constexpr (R == 4) {
        const C t0 = cadd(a[0], a[2]), t1 = csub(a[0], a[2]);
        const C t2 = cadd(a[1], a[3]), d = csub(a[1], a[3]);
        const C t3 = mkc<C>(-sign * d.y, sign * d.x);  // d * (sign i)
        a[0] = cadd(t0, t2);
        a[2] = csub(t0, t2);
        a[1] = cadd(t1, t3);
        a[3] = csub(t1, t3);
    } else {
        // odd R: p_t = a_t + a_{R-t}, m_t = a_t - a_{R-t}
        //   b_u     = a0 + sum_t [cos(th) p_t + i sign sin(th) m_t]
        //   b_{R-u} = a0 + sum_t [cos(th) p_t - i sign sin(th) m_t],  th = 2 pi t u / R
        constexpr int H = (R - 1) / 2;
        C p[H], m[H];
#pragma unroll
        for (int t = 1; t <= H; ++t) {
            p[t - 1] = cadd(a[t], a[R - t]);
            m[t - 1] = csub(a[t], a[R - t]);
        }
        const C a0 = a[0];
        C s0 = a0;
#pragma unroll
        for (int t = 0; t < H; ++t) s0 = cadd(s0, p[t]);
#pragma unroll
        for (int u = 1; u <= H; ++u) {
            C re = a0, im = mkc<C>(0, 0);
#pragma unroll
            for (int t = 1; t <= H; ++t) {
                const int idx = (t * u) % R;
                const T c = (T)(idx <= H ? oc<R>(idx - 1) : oc<R>(R - idx - 1));
                const T s = (T)(idx <= H ? os<R>(idx - 1) : -os<R>(R - idx - 1));
                re.x = fma(c, p[t - 1].x, re.x);
                re.y = fma(c, p[t - 1].y, re.y);
                im.x = fma(s, m[t - 1].x, im.x);
                im.y = fma(s, m[t - 1].y, im.y);
            }
            a[u] = mkc<C>(re.x - sign * im.y, re.y + sign * im.x);
            a[R - u] = mkc<C>(re.x + sign * im.y, re.y - sign * im.x);
        }
        a[0] = s0;
    }
}

// n / d for 0 <= n < 2^20 via M = ceil(2^40 / d) (exact, no integer divide)
__device__ __forceinline__ int fdiv(int n, unsigned long long M) {
    return (int)(((unsigned long long)(unsigned)n * M) >> 40);
}

// Thread layout of a CTA working on NL lines: line l = tid % NL, and the
// butterfly / row index advances from js in steps of JS = blockDim / NL.
struct LineMap {
    int l, js, JS;
    bool active;
    __device__ __forceinline__ explicit LineMap(int NL) {
        JS = blockDim.x / NL;
        l = threadIdx.x % NL;
        js = threadIdx.x / NL;
        active = js < JS;
    }
};

// One Stockham stage of radix R over NL lines of length P, src -> dst.
template <int R, class C>
__device__ __forceinline__ void stage(const C* __restrict__ src, C* __restrict__ dst,
                                      const C* __restrict__ tw, int P, int NL, int Ns,
                                      unsigned long long nsM, double sign, const LineMap& lm) {
    if (!lm.active) return;
    const int B = P / R;
    const int stride = P / (Ns * R);
    const int l = lm.l;
    for (int j = lm.js; j < B; j += lm.JS) {
        const int jd = fdiv(j, nsM);
        const int k = j - jd * Ns;
        C a[R];
#pragma unroll
        for (int t = 0; t < R; ++t) a[t] = src[(j + t * B) * NL + l];
        if (k) {
#pragma unroll
            for (int t = 1; t < R; ++t) {
                C w = tw[t * k * stride];  // exp(-2 pi i e / P)
                if (sign > 0) w.y = -w.y;
                a[t] = cmul(a[t], w);
            }
        }
        dft<R>(a, sign);
        const int base = jd * Ns * R + k;
#pragma unroll
        for (int u = 0; u < R; ++u) dst[(base + u * Ns) * NL + l] = a[u];
    }
}

// Full transform of NL lines (sign -1 forward, +1 inverse, unscaled) between
// the two buffers; returns the buffer holding the result.
template <class C>
__device__ __forceinline__ C* fft_lines(C* b0, C* b1, const C* tw, const FftAxis& ax, int NL,
                                              double sign, const LineMap& lm) {
    int Ns = 1;
    C* src = b0;
    C* dst = b1;
    for (int s = 0; s < ax.nst; ++s) {
        const unsigned long long M = ax.nsM[s];
        switch (ax.radix[s]) {
#define AIM_STAGE(RR) case RR: stage<RR>(src, dst, tw, ax.P, NL, Ns, M, sign, lm); break;
            AIM_STAGE(2) AIM_STAGE(3) AIM_STAGE(4) AIM_STAGE(5) AIM_STAGE(6) AIM_STAGE(7) AIM_STAGE(8)
            AIM_STAGE(9) AIM_STAGE(10) AIM_STAGE(12) AIM_STAGE(14) AIM_STAGE(15) AIM_STAGE(16)
#undef AIM_STAGE
        }
        __syncthreads();
        Ns *= ax.radix[s];
        C* t = src;
        src = dst;
        dst = t;
    }
    return src;
}

// In-place variant: every thread owns at most ONE butterfly per stage (the
// host guarantees NL * P / min_radix <= blockDim), so a stage is
// load-to-registers, barrier, compute, store -- a single shared buffer.
// One fixed register array serves every radix (kept out of the switch so it
// stays in registers across the barrier).
template <int R, class C>
__device__ __forceinline__ void ip_load(C* a, const C* __restrict__ buf, int B, int NL, int j, int l) {
#pragma unroll
    for (int t = 0; t < R; ++t) a[t] = buf[(j + t * B) * NL + l];
}

template <int R, class C>
__device__ __forceinline__ void ip_store(C* a, C* __restrict__ buf, const C* __restrict__ tw, int P,
                                         int NL, int Ns, unsigned long long nsM, double sign, int j, int l) {
    const int stride = P / (Ns * R);
    const int jd = fdiv(j, nsM);
    const int k = j - jd * Ns;
    if (k) {
#pragma unroll
        for (int t = 1; t < R; ++t) {
            C w = tw[t * k * stride];
            if (sign > 0) w.y = -w.y;
            a[t] = cmul(a[t], w);
        }
    }
    dft<R>(a, sign);
    const int base = jd * Ns * R + k;
#pragma unroll
    for (int u = 0; u < R; ++u) buf[(base + u * Ns) * NL + l] = a[u];
}

// In-place transform with runtime radices (fallback for sizes without a
// compile-time plan): every thread owns at most ONE butterfly per stage.
template <class C>
__device__ __forceinline__ void fft_lines_inplace(C* buf, const C* tw, const FftAxis& ax, int NL,
                                                  double sign, const LineMap& lm) {
    int Ns = 1;
    for (int s = 0; s < ax.nst; ++s) {
        const int R = ax.radix[s];
        const int B = ax.P / R;
        const int j = lm.js;
        const bool mine = lm.active && j < B;
        C a[16];
        if (mine) {
            switch (R) {
#define AIM_LD(RR) case RR: ip_load<RR>(a, buf, B, NL, j, lm.l); break;
                AIM_LD(2) AIM_LD(3) AIM_LD(4) AIM_LD(5) AIM_LD(6) AIM_LD(7) AIM_LD(8)
                AIM_LD(9) AIM_LD(10) AIM_LD(12) AIM_LD(14) AIM_LD(15) AIM_LD(16)
#undef AIM_LD
            }
        }
        __syncthreads();
        if (mine) {
            const unsigned long long M = ax.nsM[s];
            switch (R) {
#define AIM_ST(RR) case RR: ip_store<RR>(a, buf, tw, ax.P, NL, Ns, M, sign, j, lm.l); break;
                AIM_ST(2) AIM_ST(3) AIM_ST(4) AIM_ST(5) AIM_ST(6) AIM_ST(7) AIM_ST(8)
                AIM_ST(9) AIM_ST(10) AIM_ST(12) AIM_ST(14) AIM_ST(15) AIM_ST(16)
#undef AIM_ST
            }
        }
        __syncthreads();
        Ns *= R;
    }
}

template <int... Rs>
struct MinOf;
template <int R>
struct MinOf<R> { static constexpr int v = R; };
template <int R, int... Rs>
struct MinOf<R, Rs...> { static constexpr int v = R < MinOf<Rs...>::v ? R : MinOf<Rs...>::v; };

// ------------------------------------------- compile-time ping-pong plans
// Stockham stage src -> dst with compile-time P, Ns, R, line count NL and
// thread count T: each thread walks butterflies j = tid/NL, += T/NL (one
// butterfly live at a time: no register array survives a barrier).
template <int P, int Ns, int R, int SIGN, int NL, int T, class C>
__device__ __forceinline__ void ctp_stage(const C* src, C* dst, const C* tw) {
    constexpr Real<C> sign = SIGN;
    constexpr int B = P / R;
    constexpr int stride = P / (Ns * R);
    constexpr int JS = T / NL;
    const int l = threadIdx.x % NL;
    int j = threadIdx.x / NL;
    if (j < JS) {
#pragma unroll 1
        for (; j < B; j += JS) {
            C a[R];
            const C* sp = src + j * NL + l;   // + t * B * NL
#pragma unroll
            for (int t = 0; t < R; ++t) a[t] = sp[t * B * NL];
#ifdef AIM_BOUNDS_DEBUG
            if (!((j + (R - 1) * B) * NL + l < P * NL)) atomicCAS(&g_aim_dbg, 0, 201);
#endif
            const int jd = j / Ns;
            const int k = j - jd * Ns;
            if (Ns > 1 && k) {
#pragma unroll
                for (int t = 1; t < R; ++t) {
                    C w = tw[t * k * stride];   // exp(-2 pi i t k stride / P)
                    if (sign > 0) w.y = -w.y;
                    a[t] = cmul(a[t], w);
                }
            }
            dft<R>(a, sign);
            C* dp = dst + (jd * Ns * R + k) * NL + l;   // + u * Ns * NL
#ifdef AIM_BOUNDS_DEBUG
            if (!((jd * Ns * R + k + (R - 1) * Ns) * NL + l < P * NL)) atomicCAS(&g_aim_dbg, 0, 202);
            if (Ns > 1 && k && !((R - 1) * k * stride < P)) atomicCAS(&g_aim_dbg, 0, 203);
#endif
#pragma unroll
            for (int u = 0; u < R; ++u) dp[u * Ns * NL] = a[u];
        }
    }
    __syncthreads();
}

// Stages alternate a -> b -> a ...; returns the buffer holding the result.
template <int SIGN, int NL, int T, int P, int Ns, int R, int... Rs, class C>
__device__ __forceinline__ C* ctp_fft(C* a, C* b, const C* tw) {
    ctp_stage<P, Ns, R, SIGN, NL, T>(a, b, tw);
    if constexpr (sizeof...(Rs) > 0) return ctp_fft<SIGN, NL, T, P, Ns * R, Rs...>(b, a, tw);
    else return b;
}

template <int NL_, int T_, int P_, int... Rs>
struct CtpPlan {
    static constexpr int P = P_;
    static constexpr int NL = NL_;
    static constexpr int T = T_;
    static constexpr int min_radix = MinOf<Rs...>::v;
    template <int SIGN, class C>
    __device__ __forceinline__ static C* run(C* a, C* b, const C* tw) {
        return ctp_fft<SIGN, NL, T, P, 1, Rs...>(a, b, tw);
    }
};

// Complex elements per ping-pong buffer of one CTA (2 buffers + twiddles ~ 70 KB
// -> 3 CTAs of 256 threads per SM).
__host__ __device__ constexpr int fft_tile_capacity() { return 2304; }

}  // namespace aim
