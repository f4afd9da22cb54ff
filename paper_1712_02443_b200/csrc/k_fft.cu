// FFT convolution passes of the AIM matvec (step (ii), eq. AIM_step2,
// "the fast Fourier transform (FFT) is applied to compute
// the matrix-vector product").  Grid arrays are [4][X][Y][Z][R].
//
// fft_pass_kernel: one batched 1-D pass over a tensor viewed as [outer][L][inner]
//   * forward: zero-padding Lin -> P fused into the tile load (D11);
//   * inverse: output pruned P -> Lout at the tile store;
//   * turnaround: forward, x spectrum (octant, D12), inverse, all in smem.
// planar_yz_kernel (planar arrays, Nz small): for one (component, kx,
//   rhs chunk) plane it runs the y forward FFT (pad), the z convolution as a
//   direct Toeplitz product in registers against the 2-D spectrum
//   G2(kx, ky, |dz|), and the y inverse FFT (prune) -- one HBM round trip
//   instead of three passes over the y/z-padded grid.
#include <math.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "fft_core.cuh"

namespace aim {

template <bool INPLACE>
__global__ void __launch_bounds__(256, 2) fft_pass_kernel(FftPass p) {
    extern __shared__ double2 sm[];
    const int P = p.ax.P;
    const int TO = p.TO, TI = p.TI;
    const int NL = TO * TI;
    double2* buf = sm;
    double2* alt = INPLACE ? sm : sm + (size_t)P * NL;
    double2* tw = sm + (size_t)(INPLACE ? 1 : 2) * P * NL;

    const long long tilesI = (p.inner + TI - 1) / TI;
    const long long o0 = (long long)(blockIdx.x / tilesI) * TO;
    const long long i0 = (long long)(blockIdx.x % tilesI) * TI;
    const int to_n = (int)min((long long)TO, p.outer - o0);
    const int ti_n = (int)min((long long)TI, p.inner - i0);
    const LineMap lm(NL);
    const int o = lm.l / TI, i = lm.l - (lm.l / TI) * TI;
    const bool live = lm.active && o < to_n && i < ti_n;
    const double2* src = p.in + (o0 + o) * p.Lin * p.inner + i0 + i;

    for (int e = threadIdx.x; e < P; e += blockDim.x) tw[e] = p.ax.tw[e];
    // tile load with fused zero padding: line l = (o, i), rows j
    if (lm.active) {
        int j = lm.js;
        for (; j + 3 * lm.JS < p.Lin; j += 4 * lm.JS) {
            double2 v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
                v[q] = live ? __ldcs(src + (long long)(j + q * lm.JS) * p.inner) : make_double2(0.0, 0.0);
#pragma unroll
            for (int q = 0; q < 4; ++q) buf[(j + q * lm.JS) * NL + lm.l] = v[q];
        }
        for (; j < P; j += lm.JS)
            buf[j * NL + lm.l] = (live && j < p.Lin) ? __ldcs(src + (long long)j * p.inner) : make_double2(0.0, 0.0);
    }
    __syncthreads();

    double2* res = buf;
    if (p.mode == 1) {
        if (INPLACE) fft_lines_inplace(buf, tw, p.ax, NL, +1.0, lm);
        else res = fft_lines(buf, alt, tw, p.ax, NL, +1.0, lm);
    } else {
        if (INPLACE) fft_lines_inplace(buf, tw, p.ax, NL, -1.0, lm);
        else res = fft_lines(buf, alt, tw, p.ax, NL, -1.0, lm);
        if (p.mode == 2) {
            // x spectrum: line (o, i) belongs to outer og = (c Px + kx) Py + ky; kz = j
            if (lm.active) {
                const long long og = o0 + min(o, to_n - 1);
                const int ky = (int)(og % p.Py);
                const int kx = (int)((og / p.Py) % p.Px);
                const int ax_ = min(kx, p.Px - kx), ay = min(ky, p.Py - ky);
                const double2* g = p.spec + ((long long)ax_ * p.PyH + ay) * p.PzH;
                for (int j = lm.js; j < P; j += lm.JS) res[j * NL + lm.l] = cmul(res[j * NL + lm.l], __ldg(&g[min(j, P - j)]));
            }
            __syncthreads();
            if (INPLACE) fft_lines_inplace(res, tw, p.ax, NL, +1.0, lm);
            else res = fft_lines(res, res == buf ? alt : buf, tw, p.ax, NL, +1.0, lm);
        }
    }
    // tile store with fused pruning
    if (live) {
        double2* dst = p.out + (o0 + o) * p.Lout * p.inner + i0 + i;
        for (int j = lm.js; j < p.Lout; j += lm.JS) __stcs(dst + (long long)j * p.inner, res[j * NL + lm.l]);
    }
}

// ------------------------------------------------------------ planar y/z
constexpr int kPlanarThreads = 256;   // max; launched with min(256, Py*RC rounded to 32)
// W[4][Px][Ny][Nz][R] in place.  CTA = (plane c*Px+kx, rhs chunk r0..r0+RC).
// smem [Py][Nz*RC] (y lines indexed by l = z*RC + rl).
template <int NZ>
__global__ void __launch_bounds__(kPlanarThreads, 2) planar_yz_kernel(PlanarPass p) {
    extern __shared__ double2 sm[];
    const int Py = p.ay.P;
    const int RC = p.RC;
    const int NL = NZ * RC;
    double2* buf = sm;
    double2* tw = sm + (size_t)Py * NL;
    const int nchunk = (p.R + RC - 1) / RC;
    const long long plane = blockIdx.x / nchunk;
    const int r0 = (int)(blockIdx.x % nchunk) * RC;
    const int rc_n = min(RC, p.R - r0);
    const int kx = (int)(plane % p.Px);
    const LineMap lm(NL);
    const int z = lm.l / RC, rl = lm.l - (lm.l / RC) * RC;
    const bool live = lm.active && rl < rc_n;
    double2* W = p.W + plane * (long long)p.Ny * NZ * p.R + z * p.R + r0 + rl;   // + y * NZ * R
    const long long ystride = (long long)NZ * p.R;

    for (int e = threadIdx.x; e < Py; e += blockDim.x) tw[e] = p.ay.tw[e];
    if (lm.active) {
        int y = lm.js;
        for (; y + 3 * lm.JS < p.Ny; y += 4 * lm.JS) {
            double2 v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) v[q] = live ? __ldcs(W + (y + q * lm.JS) * ystride) : make_double2(0.0, 0.0);
#pragma unroll
            for (int q = 0; q < 4; ++q) buf[(y + q * lm.JS) * NL + lm.l] = v[q];
        }
        for (; y < Py; y += lm.JS)
            buf[y * NL + lm.l] = (live && y < p.Ny) ? __ldcs(W + y * ystride) : make_double2(0.0, 0.0);
    }
    __syncthreads();
    fft_lines_inplace(buf, tw, p.ay, NL, -1.0, lm);
    double2* res = buf;
    double2* oth = buf;   // each z line is read into registers and rewritten by one thread
    // z: out[z] = sum_z' G2(kx, ky, |z - z'|) in[z'] for every (ky, rl), one
    // line per thread, all indices compile-time (G2 row and inputs in registers),
    // symmetric Toeplitz: out[z] = g0 in[z] + sum_{d>0} g_d (in[z-d] + in[z+d]).
    const int ax_ = min(kx, p.Px - kx);
    const double2* G2 = p.spec + (long long)ax_ * p.PyH * NZ;
    for (int line = threadIdx.x; line < Py * RC; line += blockDim.x) {
        const int ky = line / RC, rr = line - (line / RC) * RC;
        const int ay = min(ky, Py - ky);
        const double2* g = G2 + (long long)ay * NZ;
        double2 gk[NZ], in[NZ];
#pragma unroll
        for (int d = 0; d < NZ; ++d) gk[d] = __ldg(&g[d]);
#pragma unroll
        for (int zz = 0; zz < NZ; ++zz) in[zz] = res[ky * NL + zz * RC + rr];
#pragma unroll
        for (int zz = 0; zz < NZ; ++zz) {
            double2 acc = cmul(gk[0], in[zz]);
#pragma unroll
            for (int d = 1; d < NZ; ++d) {
                if (zz - d < 0 && zz + d >= NZ) continue;
                double2 sum = zz - d >= 0 ? in[zz - d] : make_double2(0.0, 0.0);
                if (zz + d < NZ) sum = cadd(sum, in[zz + d]);
                acc.x = fma(gk[d].x, sum.x, fma(-gk[d].y, sum.y, acc.x));
                acc.y = fma(gk[d].x, sum.y, fma(gk[d].y, sum.x, acc.y));
            }
            oth[ky * NL + zz * RC + rr] = acc;
        }
    }
    __syncthreads();
    fft_lines_inplace(buf, tw, p.ay, NL, +1.0, lm);
    if (live)
        for (int y = lm.js; y < p.Ny; y += lm.JS) __stcs(W + y * ystride, res[y * NL + lm.l]);
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

// Radices available as one in-register butterfly (composites via fft_core's
// nested DFT).  Stage plan: fewest stages, then the larger first radix.
static const int kRadices[] = {16, 15, 14, 12, 10, 9, 8, 7, 6, 5, 4, 3, 2};

static void plan_radices(int P, std::vector<int>& best, std::vector<int>& cur) {
    if (P == 1) {
        if (best.empty() || cur.size() < best.size()) best = cur;
        return;
    }
    if (!best.empty() && cur.size() + 1 >= best.size()) return;
    for (int r : kRadices)
        if (P % r == 0) {
            cur.push_back(r);
            plan_radices(P / r, best, cur);
            cur.pop_back();
        }
}

void init_radix_twiddles() {
    static bool done[64] = {false};
    int dev = 0;
    AIM_CUDA(cudaGetDevice(&dev));
    if (dev < 64 && done[dev]) return;
    std::vector<double2> h(kRtwTotal);
    for (int R : {6, 8, 9, 10, 12, 14, 15, 16})
        for (int j = 0; j < R; ++j) {
            long double a = -2.0L * 3.141592653589793238462643383279502884L * (long double)j / (long double)R;
            h[rtw_off(R) + j] = make_double2((double)cosl(a), (double)sinl(a));
        }
    AIM_CUDA(cudaMemcpyToSymbol(c_rtw, h.data(), sizeof(double2) * kRtwTotal));
    if (dev < 64) done[dev] = true;
}

void make_fft_axis(int P, FftAxis& ax) {
    init_radix_twiddles();
    ax.P = P;
    ax.nst = 0;
    std::vector<int> best, cur;
    plan_radices(P, best, cur);
    if (P > 1 && best.empty()) throw Error(AIM_E_GRID, "FFT size not 7-smooth");
    if ((int)best.size() > kMaxStages) throw Error(AIM_E_GRID, "too many FFT stages");
    for (int r : best) ax.radix[ax.nst++] = r;
    ax.min_radix = P;
    for (int r : best) ax.min_radix = std::min(ax.min_radix, r);
    long long Ns = 1;
    for (int st = 0; st < ax.nst; ++st) {
        ax.nsM[st] = ((1ULL << 40) + (unsigned long long)Ns - 1) / (unsigned long long)Ns;
        Ns *= ax.radix[st];
    }
    std::vector<double2> h(P);
    for (int e = 0; e < P; ++e) {
        long double a = -2.0L * 3.141592653589793238462643383279502884L * (long double)e / (long double)P;
        h[e] = make_double2((double)cosl(a), (double)sinl(a));
    }
    AIM_CUDA(cudaMalloc(&ax.tw, sizeof(double2) * P));
    AIM_CUDA(cudaMemcpy(ax.tw, h.data(), sizeof(double2) * P, cudaMemcpyHostToDevice));
}

static constexpr int kFftThreads = 256;

void launch_fft_pass(const FftPass& p0, cudaStream_t s) {
    FftPass p = p0;
    const int P = p.ax.P;
    // in place when one butterfly per thread per stage suffices for >= 4 lines
    const int nl_inplace = kFftThreads * p.ax.min_radix / P;
    const bool inplace = nl_inplace >= 2;
    const int cap = std::max(fft_tile_capacity(), P);
    const int nl = inplace ? nl_inplace : std::max(1, cap / P);
    if (p.TI <= 0) {
        // TI: power of two (coalesced rows of TI*16 bytes); TO fills the tile
        long long ti = 1;
        while (ti * 2 <= std::min<long long>(p.inner, nl) && ti * 2 <= kFftThreads) ti *= 2;
        if (ti < p.inner && ti * 2 <= nl && ti * 2 <= kFftThreads) ti *= 2;  // one ragged tile is cheaper than many
        p.TI = (int)ti;
        p.TO = (int)std::max<long long>(1, std::min<long long>(p.outer, nl / p.TI));
        p.TO = std::min(p.TO, kFftThreads / p.TI);
    }
    const long long tilesI = (p.inner + p.TI - 1) / p.TI;
    const long long tilesO = (p.outer + p.TO - 1) / p.TO;
    const long long grid = tilesI * tilesO;
    if (grid <= 0) return;
    const size_t smem = sizeof(double2) * ((size_t)(inplace ? 1 : 2) * P * p.TO * p.TI + P);
    if (smem > 227 * 1024) throw Error(AIM_E_GRID, "FFT length exceeds the shared-memory tile capacity");
    static bool attr = false;
    if (!attr) {
        AIM_CUDA(cudaFuncSetAttribute(fft_pass_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        AIM_CUDA(cudaFuncSetAttribute(fft_pass_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        attr = true;
    }
    if (inplace) fft_pass_kernel<true><<<(unsigned)grid, kFftThreads, smem, s>>>(p);
    else fft_pass_kernel<false><<<(unsigned)grid, kFftThreads, smem, s>>>(p);
    note_launch("fft_pass");
}

// planar pass: one CTA holds a (Py x Nz) plane in place, one butterfly per thread per stage
bool planar_supported(int Py, int Nz, int min_radix) {
    return Nz <= kPlanarMaxNz && (long long)Nz * Py / min_radix <= kPlanarThreads && Py * Nz * 16 <= 200 * 1024;
}

void launch_planar_yz(const PlanarPass& p0, cudaStream_t s) {
    PlanarPass p = p0;
    const int Py = p.ay.P;
    const int rc_fft = (int)(kPlanarThreads * (long long)p.ay.min_radix / ((long long)Py * p.Nz));
    p.RC = std::max(1, std::min({p.R, rc_fft, kPlanarThreads / p.Nz}));
    const long long nchunk = (p.R + p.RC - 1) / p.RC;
    const long long grid = 4LL * p.Px * nchunk;
    // one z line per thread in the convolution step; NL lines for the FFT stages
    const int bfly = (int)((long long)p.Nz * p.RC * Py / p.ay.min_radix);   // butterflies per stage (max)
    const int threads = std::min(kPlanarThreads, 32 * ((std::max({bfly, Py * p.RC, p.Nz * p.RC}) + 31) / 32));
    const size_t smem = sizeof(double2) * ((size_t)Py * p.Nz * p.RC + Py);
    switch (p.Nz) {
#define PZ(NZ)                                                                                              \
    case NZ: {                                                                                              \
        static bool attr = false;                                                                           \
        if (!attr) {                                                                                        \
            AIM_CUDA(cudaFuncSetAttribute(planar_yz_kernel<NZ>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                          227 * 1024));                                                     \
            attr = true;                                                                                    \
        }                                                                                                   \
        planar_yz_kernel<NZ><<<(unsigned)grid, threads, smem, s>>>(p);                                   \
        break;                                                                                              \
    }
        PZ(1) PZ(2) PZ(3) PZ(4) PZ(5) PZ(6) PZ(7) PZ(8) PZ(9) PZ(10) PZ(11) PZ(12) PZ(13) PZ(14) PZ(15) PZ(16)
#undef PZ
        default: throw Error(AIM_E_GRID, "planar pass: Nz out of range");
    }
    note_launch("planar_yz");
}

}  // namespace aim
