// Shared-memory mixed-radix Stockham FFT passes (step (ii) of the AIM matvec,
// eq. AIM_step2: "the fast Fourier transform (FFT) is
// applied to compute the matrix-vector product").
//
// One launch = one batched 1-D pass over a tensor viewed as [outer][L][inner]:
//   * forward pass: zero-padding Lin -> P is fused into the tile load (D11);
//   * inverse pass: the output is pruned P -> Lout at the tile store;
//   * turnaround pass: forward FFT, pointwise multiply by the precomputed
//     Green's-function spectrum (octant storage, D12), inverse FFT -- all on
//     the tile in shared memory, so the spectrum product costs no extra HBM
//     round trip.
// A CTA owns TO x TI complete lines (ping-pong buffers in shared memory);
// tile loads/stores walk the `inner` index fastest, so they are contiguous
// whenever TI == inner and coalesced in TI*16-byte rows otherwise.
#include <math.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "aim_internal.cuh"

namespace aim {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }

// cos / sin (2 pi m / R), m = 1 .. (R-1)/2, for the odd radices
__constant__ double kC3[1] = {-0.5};
__constant__ double kS3[1] = {0.866025403784438596588};
__constant__ double kC5[2] = {0.309016994374947451263, -0.809016994374947451263};
__constant__ double kS5[2] = {0.951056516295153531182, 0.587785252292473137103};
__constant__ double kC7[3] = {0.623489801858733483364, -0.222520933956314392876, -0.900968867902419145999};
__constant__ double kS7[3] = {0.781831482468029803634, 0.974927912181823619342, 0.433883739117558120402};

// In-register DFT of length R, b_u = sum_t a_t exp(sign 2 pi i t u / R).
template <int R>
__device__ __forceinline__ void dft(double2* a, double sign);

template <>
__device__ __forceinline__ void dft<2>(double2* a, double) {
    double2 t = a[0];
    a[0] = cadd(t, a[1]);
    a[1] = csub(t, a[1]);
}

template <>
__device__ __forceinline__ void dft<4>(double2* a, double sign) {
    double2 t0 = cadd(a[0], a[2]), t1 = csub(a[0], a[2]);
    double2 t2 = cadd(a[1], a[3]), d = csub(a[1], a[3]);
    double2 t3 = make_double2(-sign * d.y, sign * d.x);  // d * (sign i)
    a[0] = cadd(t0, t2);
    a[2] = csub(t0, t2);
    a[1] = cadd(t1, t3);
    a[3] = csub(t1, t3);
}

// odd R: pair t with R-t:  p_t = a_t + a_{R-t}, m_t = a_t - a_{R-t}
//   b_u     = a0 + sum_t [cos(th) p_t + i sign sin(th) m_t]
//   b_{R-u} = a0 + sum_t [cos(th) p_t - i sign sin(th) m_t],  th = 2 pi t u / R
template <int R>
__device__ __forceinline__ void dft_odd(double2* a, double sign, const double* C, const double* S) {
    constexpr int H = (R - 1) / 2;
    double2 p[H], m[H];
#pragma unroll
    for (int t = 1; t <= H; ++t) {
        p[t - 1] = cadd(a[t], a[R - t]);
        m[t - 1] = csub(a[t], a[R - t]);
    }
    double2 a0 = a[0];
    double2 s0 = a0;
#pragma unroll
    for (int t = 0; t < H; ++t) s0 = cadd(s0, p[t]);
#pragma unroll
    for (int u = 1; u <= H; ++u) {
        double2 re = a0, im = make_double2(0.0, 0.0);
#pragma unroll
        for (int t = 1; t <= H; ++t) {
            int idx = (t * u) % R;            // th = 2 pi idx / R
            double c, s;
            if (idx <= H) {
                c = C[idx - 1];
                s = S[idx - 1];
            } else {
                c = C[R - idx - 1];
                s = -S[R - idx - 1];
            }
            re.x = fma(c, p[t - 1].x, re.x);
            re.y = fma(c, p[t - 1].y, re.y);
            im.x = fma(s, m[t - 1].x, im.x);
            im.y = fma(s, m[t - 1].y, im.y);
        }
        // i sign * im = sign * (-im.y, im.x)
        a[u] = make_double2(re.x - sign * im.y, re.y + sign * im.x);
        a[R - u] = make_double2(re.x + sign * im.y, re.y - sign * im.x);
    }
    a[0] = s0;
}
template <>
__device__ __forceinline__ void dft<3>(double2* a, double sign) { dft_odd<3>(a, sign, kC3, kS3); }
template <>
__device__ __forceinline__ void dft<5>(double2* a, double sign) { dft_odd<5>(a, sign, kC5, kS5); }
template <>
__device__ __forceinline__ void dft<7>(double2* a, double sign) { dft_odd<7>(a, sign, kC7, kS7); }

// One Stockham stage of radix R over NL lines of length P, src -> dst.
template <int R>
__device__ __forceinline__ void stockham_stage(const double2* __restrict__ src, double2* __restrict__ dst,
                                               const double2* __restrict__ tw, int P, int NL, int Ns,
                                               double sign) {
    const int B = P / R;
    const int stride = P / (Ns * R);
    const int total = NL * B;
    for (int b = threadIdx.x; b < total; b += blockDim.x) {
        const int l = b % NL;
        const int j = b / NL;
        const int k = j % Ns;
        double2 a[R];
#pragma unroll
        for (int t = 0; t < R; ++t) a[t] = src[(j + t * B) * NL + l];
        if (k) {
#pragma unroll
            for (int t = 1; t < R; ++t) {
                double2 w = tw[t * k * stride];  // exp(-2 pi i e / P)
                if (sign > 0) w.y = -w.y;          // inverse: conjugate
                a[t] = cmul(a[t], w);
            }
        }
        dft<R>(a, sign);
        const int base = (j / Ns) * Ns * R + k;
#pragma unroll
        for (int u = 0; u < R; ++u) dst[(base + u * Ns) * NL + l] = a[u];
    }
}

// Runs all stages; returns the buffer holding the result.
__device__ double2* run_fft(double2* b0, double2* b1, const double2* tw, const FftAxis& ax, int NL,
                            double sign) {
    int Ns = 1;
    double2* src = b0;
    double2* dst = b1;
    for (int s = 0; s < ax.nst; ++s) {
        const int R = ax.radix[s];
        switch (R) {
            case 2: stockham_stage<2>(src, dst, tw, ax.P, NL, Ns, sign); break;
            case 3: stockham_stage<3>(src, dst, tw, ax.P, NL, Ns, sign); break;
            case 4: stockham_stage<4>(src, dst, tw, ax.P, NL, Ns, sign); break;
            case 5: stockham_stage<5>(src, dst, tw, ax.P, NL, Ns, sign); break;
            case 7: stockham_stage<7>(src, dst, tw, ax.P, NL, Ns, sign); break;
        }
        __syncthreads();
        Ns *= R;
        double2* t = src;
        src = dst;
        dst = t;
    }
    return src;
}

__global__ void __launch_bounds__(512) fft_pass_kernel(FftPass p) {
    extern __shared__ double2 sm[];
    const int P = p.ax.P;
    const int TO = p.TO, TI = p.TI;
    const int NL = TO * TI;
    double2* b0 = sm;
    double2* b1 = sm + (size_t)P * NL;
    double2* tw = sm + (size_t)2 * P * NL;

    const long long tilesI = (p.inner + TI - 1) / TI;
    const long long o0 = (long long)(blockIdx.x / tilesI) * TO;
    const long long i0 = (long long)(blockIdx.x % tilesI) * TI;
    const int to_n = (int)min((long long)TO, p.outer - o0);
    const int ti_n = (int)min((long long)TI, p.inner - i0);

    for (int e = threadIdx.x; e < P; e += blockDim.x) tw[e] = p.ax.tw[e];
    // tile load with fused zero padding: element (o, j, i), i fastest
    const int tot = TO * P * TI;
    for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
        const int i = idx % TI;
        const int j = (idx / TI) % P;
        const int o = idx / (TI * P);
        double2 v = make_double2(0.0, 0.0);
        if (o < to_n && i < ti_n && j < p.Lin) v = __ldg(&p.in[((o0 + o) * p.Lin + j) * p.inner + i0 + i]);
        b0[j * NL + o * TI + i] = v;
    }
    __syncthreads();

    double2* res;
    if (p.mode == 1) {
        res = run_fft(b0, b1, tw, p.ax, NL, +1.0);
    } else {
        res = run_fft(b0, b1, tw, p.ax, NL, -1.0);
        if (p.mode == 2) {
            // x spectrum: line (o, i) belongs to outer index og = (c Px + kx) Py + ky; kz = j
            for (int idx = threadIdx.x; idx < NL * P; idx += blockDim.x) {
                const int l = idx % NL;
                const int j = idx / NL;
                const int o = l / TI;
                const long long og = o0 + min(o, to_n - 1);
                const int ky = (int)(og % p.Py);
                const int kx = (int)((og / p.Py) % p.Px);
                const int ax_ = min(kx, p.Px - kx), ay = min(ky, p.Py - ky), az = min(j, P - j);
                const double2 g = __ldg(&p.spec[((long long)ax_ * p.PyH + ay) * p.PzH + az]);
                res[idx] = cmul(res[idx], g);
            }
            __syncthreads();
            double2* other = (res == b0) ? b1 : b0;
            res = run_fft(res, other, tw, p.ax, NL, +1.0);
        }
    }
    // tile store with fused pruning
    const int tot_out = TO * p.Lout * TI;
    for (int idx = threadIdx.x; idx < tot_out; idx += blockDim.x) {
        const int i = idx % TI;
        const int j = (idx / TI) % p.Lout;
        const int o = idx / (TI * p.Lout);
        if (o < to_n && i < ti_n) p.out[((o0 + o) * p.Lout + j) * p.inner + i0 + i] = res[j * NL + o * TI + i];
    }
}

// ------------------------------------------------------------------- host
int smooth_size_at_least(int n) {
    if (n <= 1) return 1;
    for (int m = n;; ++m) {
        int r = m;
        for (int f : {2, 3, 5, 7})
            while (r % f == 0) r /= f;
        if (r == 1) return m;
    }
}

void make_fft_axis(int P, FftAxis& ax) {
    ax.P = P;
    ax.nst = 0;
    int r = P;
    while (r % 4 == 0) { ax.radix[ax.nst++] = 4; r /= 4; }
    while (r % 2 == 0) { ax.radix[ax.nst++] = 2; r /= 2; }
    for (int f : {3, 5, 7})
        while (r % f == 0) { ax.radix[ax.nst++] = f; r /= f; }
    if (r != 1 || ax.nst > kMaxStages) throw Error(AIM_E_GRID, "FFT size not 7-smooth");
    std::vector<double2> h(P);
    for (int e = 0; e < P; ++e) {
        long double a = -2.0L * 3.141592653589793238462643383279502884L * (long double)e / (long double)P;
        h[e] = make_double2((double)cosl(a), (double)sinl(a));
    }
    AIM_CUDA(cudaMalloc(&ax.tw, sizeof(double2) * P));
    AIM_CUDA(cudaMemcpy(ax.tw, h.data(), sizeof(double2) * P, cudaMemcpyHostToDevice));
}

static constexpr int kFftBudget = 6272;  // complex elements per ping-pong buffer (~100 KB)

void launch_fft_pass(const FftPass& p0, cudaStream_t s) {
    FftPass p = p0;
    const int P = p.ax.P;
    int nl = std::max(1, kFftBudget / P);
    if (p.TI <= 0) {
        long long ti = std::min<long long>(p.inner, nl);
        if (p.inner > nl && ti >= 8) ti = (ti / 8) * 8;
        p.TI = (int)ti;
        p.TO = (int)std::max<long long>(1, std::min<long long>(p.outer, nl / p.TI));
    }
    const long long tilesI = (p.inner + p.TI - 1) / p.TI;
    const long long tilesO = (p.outer + p.TO - 1) / p.TO;
    const long long grid = tilesI * tilesO;
    if (grid <= 0) return;
    const size_t smem = sizeof(double2) * ((size_t)2 * P * p.TO * p.TI + P);
    static bool attr = false;
    if (!attr) {
        AIM_CUDA(cudaFuncSetAttribute(fft_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        attr = true;
    }
    const int threads = 512;
    fft_pass_kernel<<<(unsigned)grid, threads, smem, s>>>(p);
    note_launch("fft_pass");
}

}  // namespace aim
