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
#include <cstdlib>
#include <cstring>
#include <vector>

#include "fft_core.cuh"

#ifdef AIM_BOUNDS_DEBUG
#define AIM_CHK(cond, code) do { if (!(cond)) { atomicCAS(&g_aim_dbg, 0, (code)); } } while (0)
#else
#define AIM_CHK(cond, code) do { } while (0)
#endif

namespace aim {

// ---------------------------------------------------------- async copies
// cp.async 16 B global -> shared; valid == false zero-fills the 16 bytes
// (src-size 0: nothing is read), which is how zero padding is fused in.
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc, bool valid) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gsrc), "r"(valid ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async8(void* sdst, const void* gsrc, bool valid) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gsrc), "r"(valid ? 8 : 0)
                 : "memory");
}
// one complex element (16 B complex128 / 8 B complex64), zero-filled if !valid
template <class C>
__device__ __forceinline__ void cp_async_c(C* sdst, const C* gsrc, bool valid) {
    if constexpr (sizeof(C) == 16) cp_async16(sdst, gsrc, valid);
    else cp_async8(sdst, gsrc, valid);
}
template <class C>
__device__ __forceinline__ const C* tw_of(const FftAxis& ax) {
    if constexpr (sizeof(C) == 16) return (const C*)ax.tw;
    else return (const C*)ax.tw32;
}
// Spectrum line of a turnaround pass (mode 2) for the line (outer og, inner ii):
//   spec_mode 0 (z lines): og = (c Px + kx) Py + ky, octant [ax][ay][az], line index kz;
//   spec_mode 1 (x lines of the slab path): og = c nky + kyl, ky = off + kyl,
//     kz = ii / Rin, transposed octant [ay][az][ax], line index kx.
template <class C>
__device__ __forceinline__ const C* spec_line(const FftPass& p, long long og, long long ii) {
    if (p.spec_mode == 0) {
        const int ky = (int)(og % p.Py);
        const int kx = (int)((og / p.Py) % p.Px);
        const int ax_ = min(kx, p.Px - kx), ay = min(ky, p.Py - ky);
        return ((const C*)p.spec) + ((long long)ax_ * p.PyH + ay) * p.PzH;
    }
    const int ky = p.off + (int)(og % p.nky);
    const int kz = (int)(ii / p.Rin);
    const int ay = min(ky, p.Py - ky), az = min(kz, p.Pz - kz);
    return ((const C*)p.spec) + ((long long)ay * p.PzH + az) * p.PxH;
}

__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_wait_prev() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

// Runtime radices and line count (any 7-smooth length without a compile-time
// plan; in place, one butterfly per thread per stage).
struct RtPlan {
    static constexpr int P = 0;
    static constexpr int NL = 0;
    static constexpr bool compile_time = false;
    template <int SIGN, class C>
    __device__ __forceinline__ static void run(C* buf, const C* tw, const FftAxis& ax, int NL) {
        const LineMap lm(NL);
        fft_lines_inplace(buf, tw, ax, NL, (double)SIGN, lm);
    }
};

// contiguous, balanced range of tiles for this CTA (persistent grid)
__device__ __forceinline__ void tile_range(int tiles, int& t0, int& t1) {
    const int per = tiles / (int)gridDim.x, extra = tiles % (int)gridDim.x;
    t0 = (int)blockIdx.x * per + min((int)blockIdx.x, extra);
    t1 = t0 + per + ((int)blockIdx.x < extra ? 1 : 0);
}

// Compile-time ping-pong plans (CtpPlan<lines, threads, P, radices...>) of the
// lengths the BASELINE configs use; other lengths run the runtime-radix
// kernels.  Radices <= 7: one butterfly's registers stay small.
#ifndef AIM_CT210_NL
#define AIM_CT210_NL 8
#endif
using Ct210 = CtpPlan<AIM_CT210_NL, 42 * AIM_CT210_NL, 210, 7, 6, 5>;   // x passes of C2: 8 lines (128 B rows)
using Ct24 = CtpPlan<32, 192, 24, 6, 4>;          // x passes of C1 (1 RHS): 32 lines
using Ct243 = CtpPlan<8, 216, 243, 9, 9, 3>;      // every axis of C5
using Ct486 = CtpPlan<4, 216, 486, 9, 9, 6>;      // x and y passes of C3
#ifndef AIM_CT784_NL
#define AIM_CT784_NL 4   // 4 lines of 784 per tile (x passes 0.16 -> 0.145 ms on C4)
#endif
using Ct784 = CtpPlan<AIM_CT784_NL, 112 * AIM_CT784_NL, 784, 16, 7, 7>;   // x passes of C4
using Ct210z11 = CtpPlan<11, 240, 210, 7, 6, 5>;  // planar y/z of C2, one RHS per tile
using Ct24z7 = CtpPlan<7, 64, 24, 6, 4>;          // planar y/z of C1, one RHS per tile

// ------------------------------------------------------ generic axis pass
// Persistent CTAs walk a contiguous range of (outer x inner) tiles; tile t+1
// is fetched with cp.async into the second buffer while tile t is
// transformed in place (one butterfly per thread per stage) and stored.
// Tile indices are 32-bit and advanced incrementally (no 64-bit divides:
// their call sequences pin registers and cause spills).
template <class F, int MODE, int MAXT, int MINB, class C>
__global__ void __launch_bounds__(MAXT, MINB) fft_pipe_kernel(FftPass p, int tiles) {
    extern __shared__ __align__(16) unsigned char smraw[];
    C* sm = reinterpret_cast<C*>(smraw);
    const int P = F::compile_time ? F::P : p.ax.P;
    const int TO = p.TO, TI = p.TI, NL = F::compile_time ? F::NL : TO * TI;
    C* tw = sm;
    C* const buf0 = sm + P;
    C* const buf1 = sm + P + (size_t)P * NL;
    const int outer = (int)p.outer, inner = (int)p.inner;
    const int tilesI = (inner + TI - 1) / TI;
    const LineMap lm(NL);
    const int o = lm.l / TI, i = lm.l - (lm.l / TI) * TI;
    for (int e = threadIdx.x; e < P; e += blockDim.x) tw[e] = tw_of<C>(p.ax)[e];
    int t0, t1;
    tile_range(tiles, t0, t1);
    if (t0 >= t1) return;

    // (ot, it) = tile coordinates of the tile being loaded
    int ot = t0 / tilesI, itl = t0 - (t0 / tilesI) * tilesI;
    auto issue = [&](C* buf) {
        if (!lm.active) return;
        const int oo = ot * TO + o, ii = itl * TI + i;
        const bool live = oo < outer && ii < inner;
        const C* src = ((const C*)p.in) + (live ? (long long)oo * p.Lin * inner + ii : 0);
#pragma unroll 4
        for (int j = lm.js; j < P; j += lm.JS) {
            const bool v = live && j < p.Lin;
            cp_async_c(&buf[j * NL + lm.l], v ? src + (long long)j * inner : (const C*)p.in, v);
        }
    };
    auto advance = [&]() {
        if (++itl == tilesI) { itl = 0; ++ot; }
    };
    issue(buf0);
    cp_commit();
    int cur_o = ot, cur_i = itl;   // coordinates of the tile being computed
    advance();
    for (int t = t0; t < t1; ++t) {
        const bool odd = (t - t0) & 1;
        C* buf = odd ? buf1 : buf0;
        if (t + 1 < t1) issue(odd ? buf0 : buf1);
        cp_commit();
        cp_wait_prev();
        __syncthreads();
        if constexpr (MODE == 1) {
            F::template run<+1>(buf, tw, p.ax, NL);
        } else {
            F::template run<-1>(buf, tw, p.ax, NL);
            if constexpr (MODE == 2) {
                // x spectrum: line (o, i) belongs to outer og = (c Px + kx) Py + ky; kz = j
                if (lm.active) {
                    const int og = min(cur_o * TO + o, outer - 1);
                    const C* g = spec_line<C>(p, og, min(cur_i * TI + i, inner - 1));
                    for (int j = lm.js; j < P; j += lm.JS)
                        buf[j * NL + lm.l] = cmul(buf[j * NL + lm.l], __ldg(&g[min(j, P - j)]));
                }
                __syncthreads();
                F::template run<+1>(buf, tw, p.ax, NL);
            }
        }
        // tile store with fused pruning
        const int oo = cur_o * TO + o, ii = cur_i * TI + i;
        if (lm.active && oo < outer && ii < inner) {
            C* dst = ((C*)p.out) + (long long)oo * p.Lout * inner + ii;
#pragma unroll 4
            for (int j = lm.js; j < p.Lout; j += lm.JS) __stcs(dst + (long long)j * inner, buf[j * NL + lm.l]);
        }
        cur_o = ot;
        cur_i = itl;
        advance();
        __syncthreads();
    }
}

// z step of the planar pass: out[z] = sum_z' G2(kx, ky, |z - z'|) in[z'] for
// every (ky, rl), one line per thread, all indices compile-time (inputs in
// registers), symmetric Toeplitz: out[z] = g0 in[z] + sum_{d>0} g_d (in[z-d] + in[z+d]).
template <int NZ, class C>
__device__ __forceinline__ void planar_toeplitz(C* buf, const C* g2, int Py, int RC, int NL) {
#pragma unroll 1
    for (int line = threadIdx.x; line < Py * RC; line += blockDim.x) {
        const int ky = line / RC, rr = line - (line / RC) * RC;
        const int ay = min(ky, Py - ky);
        const C* g = g2 + ay * NZ;
        C* row = buf + ky * NL + rr;   // + zz * RC
        C gk[NZ], in[NZ];
#pragma unroll
        for (int d = 0; d < NZ; ++d) gk[d] = __ldg(&g[d]);
#pragma unroll
        for (int zz = 0; zz < NZ; ++zz) in[zz] = row[zz * RC];
#pragma unroll
        for (int zz = 0; zz < NZ; ++zz) {
            C acc = cmul(gk[0], in[zz]);
#pragma unroll
            for (int d = 1; d < NZ; ++d) {
                if (zz - d < 0 && zz + d >= NZ) continue;
                C sum = zz - d >= 0 ? in[zz - d] : mkc<C>(0, 0);
                if (zz + d < NZ) sum = zz - d >= 0 ? cadd(sum, in[zz + d]) : in[zz + d];
                const C gd = gk[d];
                acc.x = fma(gd.x, sum.x, fma(-gd.y, sum.y, acc.x));
                acc.y = fma(gd.x, sum.y, fma(gd.y, sum.x, acc.y));
            }
            row[zz * RC] = acc;
        }
    }
}

// --------------------------------------------- compile-time pass kernels
// Persistent CTAs, three tile buffers: X holds the tile being transformed, Y
// is the ping-pong scratch, Z receives the next tile by cp.async; X and Z
// swap after every tile.  All sizes compile-time (F::P, F::NL, F::T).
template <class F, int MODE, int MINB, class C, bool TAB = false>
__global__ void __launch_bounds__(F::T, MINB) fft_ct_kernel(FftPass p, int tiles) {
    constexpr int P = F::P, NL = F::NL, T = F::T, JS = T / NL;
    extern __shared__ __align__(16) unsigned char smraw[];
    C* sm = reinterpret_cast<C*>(smraw);
    C* tw = sm;
    C* X = sm + P;
    C* Y = X + P * NL;
    C* Z = Y + P * NL;
    const int TI = p.TI;
    const int outer = (int)p.outer, inner = (int)p.inner;
    const int tilesI = (inner + TI - 1) / TI;
    const int l = threadIdx.x % NL, js = threadIdx.x / NL;
    const bool act = js < JS;
    const int o = l / TI, i = l - (l / TI) * TI;
    for (int e = threadIdx.x; e < P; e += T) tw[e] = tw_of<C>(p.ax)[e];
    int t0, t1;
    tile_range(tiles, t0, t1);
    if (t0 >= t1) return;
    int ot = t0 / tilesI, itl = t0 - (t0 / tilesI) * tilesI;
    auto issue = [&](C* buf) {
        if (!act) return;
        const int oo = ot * (NL / TI) + o, ii = itl * TI + i;
        const bool live = oo < outer && ii < inner;
        const bool tin = TAB && p.jin != nullptr;   // lines addressed through the jin table (fused unpack)
        const C* src = ((const C*)p.in) + (live ? (long long)oo * (tin ? 1 : p.Lin) * inner + ii : 0);
#pragma unroll 2
        for (int j = js; j < P; j += JS) {
            const bool v = live && j < p.Lin;
            long long jo = (long long)j * inner;
            if constexpr (TAB) { if (tin && v) jo = __ldg(&p.jin[j]); }
            cp_async_c(&buf[j * NL + l], v ? src + jo : (const C*)p.in, v);
        }
    };
    auto advance = [&]() {
        if (++itl == tilesI) { itl = 0; ++ot; }
    };
    issue(X);
    cp_commit();
    int cur_o = ot, cur_i = itl;
    advance();
    for (int t = t0; t < t1; ++t) {
        if (t + 1 < t1) issue(Z);
        cp_commit();
        cp_wait_prev();
        __syncthreads();
        C* res;
        if constexpr (MODE == 1) {
            res = F::template run<+1>(X, Y, tw);
        } else {
            res = F::template run<-1>(X, Y, tw);
            if constexpr (MODE == 2) {
                if (act) {
                    const int og = min(cur_o * (NL / TI) + o, outer - 1);
                    const C* g = spec_line<C>(p, og, min(cur_i * TI + i, inner - 1));
                    for (int j = js; j < P; j += JS) res[j * NL + l] = cmul(res[j * NL + l], __ldg(&g[min(j, P - j)]));
                }
                __syncthreads();
                res = F::template run<+1>(res, res == X ? Y : X, tw);
            }
        }
        const int oo = cur_o * (NL / TI) + o, ii = cur_i * TI + i;
        if (act && oo < outer && ii < inner) {
            if constexpr (TAB) {
                if (p.jout != nullptr) {      // fused pack: line j goes to its owner's block
                    C* dst = ((C*)p.out) + (long long)oo * inner + ii;
#pragma unroll 2
                    for (int j = js; j < p.Lout; j += JS) __stcs(dst + __ldg(&p.jout[j]), res[j * NL + l]);
                } else {
                    C* dst = ((C*)p.out) + (long long)oo * p.Lout * inner + ii;
#pragma unroll 2
                    for (int j = js; j < p.Lout; j += JS) __stcs(dst + (long long)j * inner, res[j * NL + l]);
                }
            } else {
                C* dst = ((C*)p.out) + (long long)oo * p.Lout * inner + ii;
#pragma unroll 2
                for (int j = js; j < p.Lout; j += JS) __stcs(dst + (long long)j * inner, res[j * NL + l]);
            }
        }
        cur_o = ot;
        cur_i = itl;
        advance();
        C* tmp = X;
        X = Z;
        Z = tmp;
        __syncthreads();
    }
}

// Planar y/z pass with a compile-time plan: persistent CTAs, three tile
// buffers (X being transformed, Y ping-pong scratch, Z receiving the next
// tile by cp.async); the twiddles and the G2 slice are read through L1
// (__ldg) so two CTAs fit per SM (barrier stalls of one overlap the other).
template <int NZ, class F, int MINB, class C>
__global__ void __launch_bounds__(F::T, MINB) planar_ct_kernel(PlanarPass p, int tiles) {
    constexpr int Py = F::P, NL = F::NL, T = F::T, JS = T / NL;
    static_assert(NL == NZ, "one RHS per tile");
    extern __shared__ __align__(16) unsigned char smraw[];
    C* sm = reinterpret_cast<C*>(smraw);
    C* X = sm;
    C* Y = X + Py * NL;
    C* Z = Y + Py * NL;
    const C* tw = tw_of<C>(p.ay);
    const int nchunk = p.R;
    const int l = threadIdx.x % NL, js = threadIdx.x / NL;   // l = z
    const bool act = js < JS;
    const int ystride = NZ * p.R;
    int t0, t1;
    tile_range(tiles, t0, t1);
    if (t0 >= t1) return;
    int lkx = t0 / (4 * nchunk), lc = (t0 / nchunk) % 4, lch = t0 % nchunk;
    auto base_of = [&](int kx, int c, int r) -> C* {
        const long long plane = (long long)c * p.Px + kx;
        return ((C*)p.W) + plane * p.Ny * ystride + l * p.R + r;   // + y * ystride
    };
    auto issue = [&](C* buf) {
        if (!act) return;
        const C* src = base_of(lkx, lc, lch);
#pragma unroll 2
        for (int y = js; y < Py; y += JS) {
            const bool v = y < p.Ny;
            cp_async_c(&buf[y * NL + l], v ? src + y * ystride : (const C*)p.W, v);
        }
    };
    auto advance = [&]() {
        if (++lch == nchunk) {
            lch = 0;
            if (++lc == 4) { lc = 0; ++lkx; }
        }
    };
    issue(X);
    cp_commit();
    int ckx = lkx, cc = lc, cch = lch;
    advance();
    for (int t = t0; t < t1; ++t) {
        if (t + 1 < t1) issue(Z);
        cp_commit();
        cp_wait_prev();
        __syncthreads();
        const int kg = ckx + p.off;   // global index of the outer (spectral) axis
        const int ax_ = min(kg, p.Pfold - kg);
        const C* g2 = ((const C*)p.spec) + (long long)ax_ * p.PyH * NZ;
        C* res = F::template run<-1>(X, Y, tw);
        planar_toeplitz<NZ>(res, g2, Py, 1, NL);
        __syncthreads();
        res = F::template run<+1>(res, res == X ? Y : X, tw);
        if (act) {
            C* dst = base_of(ckx, cc, cch);
#pragma unroll 2
            for (int y = js; y < p.Ny; y += JS) __stcs(dst + y * ystride, res[y * NL + l]);
        }
        ckx = lkx; cc = lc; cch = lch;
        advance();
        C* tmp = X;
        X = Z;
        Z = tmp;
        __syncthreads();
    }
}

// Four-step planar y/z pass (complex128, Py = N1 N2): every half-warp owns one
// z line of the (kx, component, rhs) tile and transforms it in registers,
//   forward  step 1: lane n2 < N2: DFT_N1 over x[N2 n1 + n2], x w^(n2 k1) -> row N2 k1 + n2
//            step 2: lane k1 < N1: DFT_N2 over rows N2 k1 + n2       -> X[k1 + N1 k2]
// (each step reads and writes only the half-warp's own column of the [y][z]
// tile; __syncwarp separates the steps), then the CTA-wide z Toeplitz x G2
// (spectrum slice of this kx staged in shared memory), then the same two steps
// with conjugate twiddles and the pruned output (y < Ny) stored straight from
// registers.  Versus the Stockham stage kernel: 2 register passes instead of 3
// shared-memory stages per direction and no CTA barrier inside the FFTs.
// Persistent CTAs; the next tile is fetched by cp.async into a second buffer.
template <int NZ, int N1, int N2, int NW>
__global__ void __launch_bounds__(32 * NW, 2) planar4_kernel(PlanarPass p, int tiles) {
    constexpr int Py = N1 * N2, T = 32 * NW;
    static_assert(2 * NW >= NZ, "one z line per half-warp");
    constexpr int PyH = Py / 2 + 1;
    static_assert(N1 <= 16 && N2 <= 16, "register radices");
    extern __shared__ __align__(16) unsigned char smraw[];
    double2* bufA = reinterpret_cast<double2*>(smraw);
    double2* bufB = bufA + Py * NZ;
    double2* g2s = bufB + Py * NZ;        // [PyH][NZ] spectrum slice of the current kx
    double2* tws = g2s + PyH * NZ;        // [Py] exp(-2 pi i e / Py)
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int z = 2 * w + (lane >> 4), h = lane & 15;
    const bool zl = z < NZ;
    const int nchunk = p.R;
    const int ystride = NZ * p.R;
    for (int e = threadIdx.x; e < Py; e += T) tws[e] = p.ay.tw[e];
    int t0, t1;
    tile_range(tiles, t0, t1);
    if (t0 >= t1) return;
    int lkx = t0 / (4 * nchunk), lc = (t0 / nchunk) % 4, lch = t0 % nchunk;
    auto base_of = [&](int kx, int c, int r) -> double2* {
        const long long plane = (long long)c * p.Px + kx;
        return ((double2*)p.W) + plane * p.Ny * ystride + r;   // + y * ystride + z * R
    };
    // tile load: [y][z] rows, zero rows y >= Ny (the padding), coalesced over z
    auto issue = [&](double2* buf) {
        const double2* src = base_of(lkx, lc, lch);
        for (int e = threadIdx.x; e < Py * NZ; e += T) {
            const int yy = e / NZ, zz = e - (e / NZ) * NZ;
            const bool v = yy < p.Ny;
            cp_async_c(&buf[e], v ? src + (long long)yy * ystride + zz * p.R : (const double2*)p.W, v);
        }
    };
    auto advance = [&]() {
        if (++lch == nchunk) {
            lch = 0;
            if (++lc == 4) { lc = 0; ++lkx; }
        }
    };
    double2* X = bufA;
    double2* Z = bufB;
    issue(X);
    cp_commit();
    int ckx = lkx, cc = lc, cch = lch;
    int g2kx = -1;
    advance();
    for (int t = t0; t < t1; ++t) {
        if (t + 1 < t1) issue(Z);
        cp_commit();
        const int kg = ckx + p.off;
        const int ax_ = min(kg, p.Pfold - kg);
        if (ax_ != g2kx) {   // stage the spectrum slice of this kx (uniform across the CTA)
            const double2* g2 = ((const double2*)p.spec) + (long long)ax_ * PyH * NZ;
            for (int e = threadIdx.x; e < PyH * NZ; e += T) g2s[e] = __ldg(&g2[e]);
            g2kx = ax_;
        }
        cp_wait_prev();
        __syncthreads();
        double2* col = X + z;   // this half-warp's column: element y at col[y * NZ]
        // ---- forward, step 1
        if (zl && h < N2) {
            double2 a[N1];
#pragma unroll
            for (int n1 = 0; n1 < N1; ++n1) a[n1] = col[(N2 * n1 + h) * NZ];
            dft<N1>(a, -1.0);
#pragma unroll
            for (int k1 = 1; k1 < N1; ++k1) a[k1] = cmul(a[k1], tws[h * k1]);
#pragma unroll
            for (int k1 = 0; k1 < N1; ++k1) col[(N2 * k1 + h) * NZ] = a[k1];
        }
        __syncwarp();
        // ---- forward, step 2
        {
            double2 b[N2];
            const bool act = zl && h < N1;
            if (act) {
#pragma unroll
                for (int n2 = 0; n2 < N2; ++n2) b[n2] = col[(N2 * h + n2) * NZ];
                dft<N2>(b, -1.0);
            }
            __syncwarp();
            if (act) {
#pragma unroll
                for (int k2 = 0; k2 < N2; ++k2) col[(h + N1 * k2) * NZ] = b[k2];
            }
        }
        __syncthreads();
        // ---- z Toeplitz against G2(kx, ky, |dz|)
        for (int ky = threadIdx.x; ky < Py; ky += T) {
            const int ay = min(ky, Py - ky);
            const double2* g = g2s + ay * NZ;
            double2* row = X + ky * NZ;
            double2 gk[NZ], in[NZ];
#pragma unroll
            for (int d = 0; d < NZ; ++d) gk[d] = g[d];
#pragma unroll
            for (int zz = 0; zz < NZ; ++zz) in[zz] = row[zz];
#pragma unroll
            for (int zz = 0; zz < NZ; ++zz) {
                double2 acc = cmul(gk[0], in[zz]);
#pragma unroll
                for (int d = 1; d < NZ; ++d) {
                    if (zz - d < 0 && zz + d >= NZ) continue;
                    double2 sum = zz - d >= 0 ? in[zz - d] : make_double2(0.0, 0.0);
                    if (zz + d < NZ) sum = zz - d >= 0 ? cadd(sum, in[zz + d]) : in[zz + d];
                    const double2 gd = gk[d];
                    acc.x = fma(gd.x, sum.x, fma(-gd.y, sum.y, acc.x));
                    acc.y = fma(gd.x, sum.y, fma(gd.y, sum.x, acc.y));
                }
                row[zz] = acc;
            }
        }
        __syncthreads();
        // ---- inverse, step 1
        if (zl && h < N2) {
            double2 a[N1];
#pragma unroll
            for (int n1 = 0; n1 < N1; ++n1) a[n1] = col[(N2 * n1 + h) * NZ];
            dft<N1>(a, +1.0);
#pragma unroll
            for (int k1 = 1; k1 < N1; ++k1) {
                double2 tw = tws[h * k1];
                tw.y = -tw.y;
                a[k1] = cmul(a[k1], tw);
            }
#pragma unroll
            for (int k1 = 0; k1 < N1; ++k1) col[(N2 * k1 + h) * NZ] = a[k1];
        }
        __syncwarp();
        // ---- inverse, step 2 and the pruned store (y = k1 + N1 k2 < Ny)
        if (zl && h < N1) {
            double2 b[N2];
#pragma unroll
            for (int n2 = 0; n2 < N2; ++n2) b[n2] = col[(N2 * h + n2) * NZ];
            dft<N2>(b, +1.0);
            double2* dst = base_of(ckx, cc, cch) + z * p.R;
#pragma unroll
            for (int k2 = 0; k2 < N2; ++k2) {
                const int yy = h + N1 * k2;
                if (yy < p.Ny) __stcs(dst + (long long)yy * ystride, b[k2]);
            }
        }
        ckx = lkx; cc = lc; cch = lch;
        advance();
        double2* tmp = X;
        X = Z;
        Z = tmp;
        __syncthreads();
    }
}

// Ping-pong fallback (lines too long for one butterfly per thread): one tile
// per CTA, two buffers.
template <class C>
__global__ void __launch_bounds__(256, 2) fft_pp_kernel(FftPass p) {
    extern __shared__ __align__(16) unsigned char smraw[];
    C* sm = reinterpret_cast<C*>(smraw);
    const int P = p.ax.P;
    const int TO = p.TO, TI = p.TI;
    const int NL = TO * TI;
    C* buf = sm;
    C* alt = sm + (size_t)P * NL;
    C* tw = sm + (size_t)2 * P * NL;

    const long long tilesI = (p.inner + TI - 1) / TI;
    const long long o0 = (long long)(blockIdx.x / tilesI) * TO;
    const long long i0 = (long long)(blockIdx.x % tilesI) * TI;
    const int to_n = (int)min((long long)TO, p.outer - o0);
    const int ti_n = (int)min((long long)TI, p.inner - i0);
    const LineMap lm(NL);
    const int o = lm.l / TI, i = lm.l - (lm.l / TI) * TI;
    const bool live = lm.active && o < to_n && i < ti_n;
    const C* src = ((const C*)p.in) + (o0 + o) * p.Lin * p.inner + i0 + i;

    for (int e = threadIdx.x; e < P; e += blockDim.x) tw[e] = tw_of<C>(p.ax)[e];
    if (lm.active)
        for (int j = lm.js; j < P; j += lm.JS) {
            const bool v = live && j < p.Lin;
            cp_async_c(&buf[j * NL + lm.l], v ? src + (long long)j * p.inner : (const C*)p.in, v);
        }
    cp_commit();
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();

    C* res = buf;
    if (p.mode == 1) {
        res = fft_lines(buf, alt, tw, p.ax, NL, +1.0, lm);
    } else {
        res = fft_lines(buf, alt, tw, p.ax, NL, -1.0, lm);
        if (p.mode == 2) {
            if (lm.active) {
                const long long og = o0 + min(o, to_n - 1);
                const C* g = spec_line<C>(p, og, i0 + min(i, ti_n - 1));
                for (int j = lm.js; j < P; j += lm.JS) res[j * NL + lm.l] = cmul(res[j * NL + lm.l], __ldg(&g[min(j, P - j)]));
            }
            __syncthreads();
            res = fft_lines(res, res == buf ? alt : buf, tw, p.ax, NL, +1.0, lm);
        }
    }
    if (live) {
        C* dst = ((C*)p.out) + (o0 + o) * p.Lout * p.inner + i0 + i;
        for (int j = lm.js; j < p.Lout; j += lm.JS) __stcs(dst + (long long)j * p.inner, res[j * NL + lm.l]);
    }
}

// ------------------------------------------------------------ planar y/z
constexpr int kPlanarThreads = 256;   // max; launched with >= one butterfly per line element / min radix
// W[4][Px][Ny][Nz][R] in place.  Tile = (plane c*Px+kx, rhs chunk r0..r0+RC),
// ordered kx-major (a CTA's tile range touches the G2 slices of one or two kx,
// read through L1).  smem: twiddles [Py], two tile buffers [Py][NZ*RC]
// (y lines indexed by l = z*RC + rl).
template <int NZ, class F, int MAXT, int MINB, class C>
__global__ void __launch_bounds__(MAXT, MINB) planar_yz_kernel(PlanarPass p, int tiles) {
    extern __shared__ __align__(16) unsigned char smraw[];
    C* sm = reinterpret_cast<C*>(smraw);
    const int Py = F::compile_time ? F::P : p.ay.P;
    const int RC = F::compile_time ? 1 : p.RC;
    const int NL = NZ * RC;
    C* tw = sm;
    C* const buf0 = sm + Py;
    C* const buf1 = buf0 + (size_t)Py * NL;
    const int nchunk = (p.R + RC - 1) / RC;
    const LineMap lm(NL);
    const int z = lm.l / RC, rl = lm.l - (lm.l / RC) * RC;
    const int ystride = NZ * p.R;
    for (int e = threadIdx.x; e < Py; e += blockDim.x) tw[e] = tw_of<C>(p.ay)[e];
    int t0, t1;
    tile_range(tiles, t0, t1);
    if (t0 >= t1) return;

    // tile t -> (kx, c, chunk) = (t / (4 nchunk), (t / nchunk) % 4, t % nchunk); advanced incrementally
    int lkx = t0 / (4 * nchunk), lc = (t0 / nchunk) % 4, lch = t0 % nchunk;
    auto base_of = [&](int kx, int c, int ch, bool& live) -> C* {
        const int r0 = ch * RC;
        live = lm.active && r0 + rl < p.R;
        const long long plane = (long long)c * p.Px + kx;
        return ((C*)p.W) + plane * p.Ny * ystride + z * p.R + r0 + rl;   // + y * ystride
    };
    auto issue = [&](C* buf) {
        if (!lm.active) return;
        bool live;
        const C* src = base_of(lkx, lc, lch, live);
#pragma unroll 4
        for (int y = lm.js; y < Py; y += lm.JS) {
            const bool v = live && y < p.Ny;
            cp_async_c(&buf[y * NL + lm.l], v ? src + y * ystride : (const C*)p.W, v);
        }
    };
    auto advance = [&]() {
        if (++lch == nchunk) {
            lch = 0;
            if (++lc == 4) { lc = 0; ++lkx; }
        }
    };
    issue(buf0);
    cp_commit();
    int ckx = lkx, cc = lc, cch = lch;   // tile being computed
    advance();
    for (int t = t0; t < t1; ++t) {
        const bool odd = (t - t0) & 1;
        C* buf = odd ? buf1 : buf0;
        if (t + 1 < t1) issue(odd ? buf0 : buf1);
        cp_commit();
        cp_wait_prev();
        const int kg = ckx + p.off;   // global index of the outer (spectral) axis
        const int ax_ = min(kg, p.Pfold - kg);
        const C* g2 = ((const C*)p.spec) + (long long)ax_ * p.PyH * NZ;   // G2 slice of this kx (read through L1)
        __syncthreads();
        F::template run<-1>(buf, tw, p.ay, NL);
        planar_toeplitz<NZ>(buf, g2, Py, RC, NL);
        __syncthreads();
        F::template run<+1>(buf, tw, p.ay, NL);
        bool live;
        C* dst = base_of(ckx, cc, cch, live);
        if (live) {
#pragma unroll 4
            for (int y = lm.js; y < p.Ny; y += lm.JS) __stcs(dst + y * ystride, buf[y * NL + lm.l]);
        }
        ckx = lkx; cc = lc; cch = lch;
        advance();
        __syncthreads();
    }
}

// ------------------------------------------------------- z Toeplitz (mode 2)
// Thread per z line (component, a, b, rhs) of W[4][A][B][NZ][R]:
//   out[z] = sum_z' G2(kx, ky, |z - z'|) in[z'],  symmetric form
//   out[z] = g0 in[z] + sum_{d>0} g_d (in[z-d] + in[z+d]).
// The line's NZ values are one contiguous run for R = 1 (the GMRES case).
template <int NZ, class C>
__global__ void __launch_bounds__(128) ztoeplitz_kernel(C* __restrict__ W, long long lines, int A, int B, int R,
                                                        int kx_is_a, int off, int Px, int Py,
                                                        const C* __restrict__ spec) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= lines) return;
    const int r = (int)(t % R);
    long long q = t / R;
    const int b = (int)(q % B);
    q /= B;
    const int a = (int)(q % A);
    const int c = (int)(q / A);
    const int kx = kx_is_a ? a : b, ky = kx_is_a ? b + off : a + off;
    const int ax_ = min(kx, Px - kx), ay = min(ky, Py - ky);
    const C* g = spec + ((long long)ax_ * (Py / 2 + 1) + ay) * NZ;
    C* row = W + (((long long)c * A + a) * B + b) * NZ * R + r;
    C in[NZ];
#pragma unroll
    for (int z = 0; z < NZ; ++z) in[z] = row[(long long)z * R];
#pragma unroll
    for (int z = 0; z < NZ; ++z) {
        C acc = cmul(__ldg(&g[0]), in[z]);
#pragma unroll
        for (int d = 1; d < NZ; ++d) {
            if (z - d < 0 && z + d >= NZ) continue;
            C sum = z - d >= 0 ? in[z - d] : mkc<C>(0, 0);
            if (z + d < NZ) sum = z - d >= 0 ? cadd(sum, in[z + d]) : in[z + d];
            const C gd = __ldg(&g[d]);
            acc.x = fma(gd.x, sum.x, fma(-gd.y, sum.y, acc.x));
            acc.y = fma(gd.x, sum.y, fma(gd.y, sum.x, acc.y));
        }
        __stcs(&row[(long long)z * R], acc);
    }
}

template <class C>
static void launch_ztoeplitz_t(C* W, int A, int B, int Nz, int R, int kx_is_a, int off, int Px, int Py,
                               const C* spec, cudaStream_t s) {
    const long long lines = 4LL * A * B * R;
    if (lines <= 0) return;
    const unsigned grid = (unsigned)((lines + 127) / 128);
    switch (Nz) {
#define ZT(NZ) case NZ: ztoeplitz_kernel<NZ, C><<<grid, 128, 0, s>>>(W, lines, A, B, R, kx_is_a, off, Px, Py, spec); break;
        ZT(1) ZT(2) ZT(3) ZT(4) ZT(5) ZT(6) ZT(7) ZT(8) ZT(9) ZT(10) ZT(11) ZT(12) ZT(13) ZT(14) ZT(15) ZT(16)
#undef ZT
        default: throw Error(AIM_E_GRID, "z Toeplitz: Nz out of range");
    }
}

void launch_ztoeplitz(void* W, int prec, int A, int B, int Nz, int R, int kx_is_a, int off, int Px, int Py,
                      const void* spec, cudaStream_t s) {
    if (prec == 1) launch_ztoeplitz_t((float2*)W, A, B, Nz, R, kx_is_a, off, Px, Py, (const float2*)spec, s);
    else launch_ztoeplitz_t((double2*)W, A, B, Nz, R, kx_is_a, off, Px, Py, (const double2*)spec, s);
    note_launch("ztoeplitz");
}

#include "ymode2.cuh"

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

static int min_of(const std::vector<int>& v) {
    int m = 1 << 30;
    for (int r : v) m = std::min(m, r);
    return m;
}

// fewest stages, then the largest smallest radix (fewer threads idle in the
// in-place kernels), then the first found (larger first radix)
static void plan_radices(int P, std::vector<int>& best, std::vector<int>& cur) {
    if (P == 1) {
        if (best.empty() || cur.size() < best.size() || (cur.size() == best.size() && min_of(cur) > min_of(best)))
            best = cur;
        return;
    }
    if (!best.empty() && cur.size() + 1 > best.size()) return;
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
    for (int R : {6, 8, 9, 10, 12, 14, 15, 16, 28})
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
    h2d(ax.tw, h.data(), sizeof(double2) * P, 0);
    std::vector<float2> h32(P);
    for (int e = 0; e < P; ++e) h32[e] = make_float2((float)h[e].x, (float)h[e].y);
    AIM_CUDA(cudaMalloc(&ax.tw32, sizeof(float2) * P));
    h2d(ax.tw32, h32.data(), sizeof(float2) * P, 0);
}

static constexpr int kFftThreads = 256;

static int sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        AIM_CUDA(cudaGetDevice(&dev));
        AIM_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    }
    return n;
}

// Opt a kernel into the full 227 KB of dynamic shared memory (once per kernel
// and device; kernels are distinguished by address, not by signature).
template <class K>
static void ensure_smem_attr(K kernel) {
    static std::vector<std::pair<const void*, int>> done;
    int dev = 0;
    AIM_CUDA(cudaGetDevice(&dev));
    const void* key = (const void*)kernel;
    for (auto& d : done)
        if (d.first == key && d.second == dev) return;
    AIM_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    // with the near SpMV beside the FFT (k_near_stream.cu) every SM stays in
    // its largest shared-memory configuration, so both CTAs fit at once
    if (smem_carveout_max())
        AIM_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    done.emplace_back(key, dev);
}

template <class K>
static long long persistent_grid(K kernel, int threads, size_t smem, long long tiles) {
    if (tiles >= (1LL << 31)) throw Error(AIM_E_GRID, "FFT pass: tile count exceeds 2^31");
    int per = 0;
    AIM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, threads, smem));
    return std::max(1LL, std::min(tiles, (long long)std::max(1, per) * sm_count()));
}

// Tile shape for TI x TO lines of a pass with nl lines available.
static void tile_shape(FftPass& p, int nl) {
    long long ti = 1;
    while (ti * 2 <= std::min<long long>(p.inner, nl) && ti * 2 <= kFftThreads) ti *= 2;
    if (ti < p.inner && ti * 2 <= nl && ti * 2 <= kFftThreads) ti *= 2;  // one ragged tile is cheaper than many
    p.TI = (int)ti;
    p.TO = (int)std::max<long long>(1, std::min<long long>(p.outer, nl / p.TI));
    p.TO = std::min(p.TO, std::max(1, nl / p.TI));
}

template <class C, class K>
static void launch_pipe(K kern, const FftPass& p, int threads, cudaStream_t s) {
    const int P = p.ax.P;
    const long long tiles = ((p.inner + p.TI - 1) / p.TI) * ((p.outer + p.TO - 1) / p.TO);
    if (tiles <= 0) return;
    const size_t smem = sizeof(C) * ((size_t)2 * P * p.TO * p.TI + P);
    if (smem > 227 * 1024) throw Error(AIM_E_GRID, "FFT length exceeds the shared-memory tile capacity");
    ensure_smem_attr(kern);
    const long long grid = persistent_grid(kern, threads, smem, tiles);
    kern<<<(unsigned)grid, threads, smem, s>>>(p, (int)tiles);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        throw Error(AIM_E_CUDA, "fft_pipe_kernel P=" + std::to_string(P) + " NL=" + std::to_string(p.TO * p.TI) +
                                    " threads=" + std::to_string(threads) + " grid=" + std::to_string(grid) +
                                    " smem=" + std::to_string(smem) + ": " + cudaGetErrorString(e));
}

template <class C, class F, int MINB>
static bool try_ct_pass(FftPass p, cudaStream_t s) {
    if (p.ax.P != F::P || p.TI > 0) return false;
    // F::NL lines: TI = the largest power of two <= inner dividing NL, TO = NL / TI
    int ti = 1;
    while (F::NL % (ti * 2) == 0 && ti * 2 <= p.inner) ti *= 2;
    if (F::NL / ti > p.outer) return false;
    p.TI = ti;
    p.TO = F::NL / ti;
    const long long tiles = ((p.inner + p.TI - 1) / p.TI) * ((p.outer + p.TO - 1) / p.TO);
    const size_t smem = sizeof(C) * ((size_t)3 * F::P * F::NL + F::P);
    auto go = [&](auto kern) {
        ensure_smem_attr(kern);
        const long long grid = persistent_grid(kern, F::T, smem, tiles);
        kern<<<(unsigned)grid, F::T, smem, s>>>(p, (int)tiles);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess)
            throw Error(AIM_E_CUDA, "fft_ct_kernel P=" + std::to_string(F::P) + ": " + cudaGetErrorString(e));
    };
    if (p.jin || p.jout) {
        // table-addressed lines: complex128, forward/inverse, the planar configs' lengths
        if constexpr (sizeof(C) == 16 && (F::P == 210 || F::P == 784)) {
            if (p.mode == 0) go(fft_ct_kernel<F, 0, MINB, C, true>);
            else if (p.mode == 1) go(fft_ct_kernel<F, 1, MINB, C, true>);
            else return false;
            return true;
        } else {
            return false;
        }
    }
    if (p.mode == 0) go(fft_ct_kernel<F, 0, MINB, C>);
    else if (p.mode == 1) go(fft_ct_kernel<F, 1, MINB, C>);
    else go(fft_ct_kernel<F, 2, MINB, C>);
    return true;
}

template <class C>
static void launch_fft_pass_t(FftPass p, cudaStream_t s) {
    const int P = p.ax.P;
    const char* ce = getenv("AIM_FFT_NOCT");   // A/B timing: skip the compile-time plans
    if (!(ce && ce[0] == '1') &&
        (try_ct_pass<C, Ct210, 2>(p, s) || try_ct_pass<C, Ct24, 2>(p, s) || try_ct_pass<C, Ct243, 2>(p, s) ||
         try_ct_pass<C, Ct486, 2>(p, s) || try_ct_pass<C, Ct784, (AIM_CT784_NL > 2 ? 1 : 2)>(p, s)))
        return;
    // runtime radices: in place when one butterfly per thread per stage suffices for >= 2 lines
    const int nl_inplace = kFftThreads * p.ax.min_radix / P;
    // The ping-pong kernel (several butterflies per thread, up to
    // fft_tile_capacity() elements per tile, one tile per CTA) beats the
    // persistent in-place kernel on every measured size (C3 FFT 0.98 -> 0.60 ms,
    // C4 1.93 -> 1.67, C5 5.70 -> 2.05 ms: the in-place kernel's one butterfly
    // per thread limits a tile to 256 * min_radix / P lines, 3 for P = 243).
    // AIM_FFT_INPLACE=1 restores the in-place kernel (A/B timing).
    const char* fe = getenv("AIM_FFT_INPLACE");
    const bool inplace = nl_inplace >= 2 && fe && fe[0] == '1';
    const int cap = std::max(fft_tile_capacity(), P);
    if (p.TI <= 0) tile_shape(p, inplace ? nl_inplace : std::max(1, cap / P));
    if (inplace) {
        if (p.mode == 0) launch_pipe<C>(fft_pipe_kernel<RtPlan, 0, kFftThreads, 2, C>, p, kFftThreads, s);
        else if (p.mode == 1) launch_pipe<C>(fft_pipe_kernel<RtPlan, 1, kFftThreads, 2, C>, p, kFftThreads, s);
        else launch_pipe<C>(fft_pipe_kernel<RtPlan, 2, kFftThreads, 2, C>, p, kFftThreads, s);
    } else {
        const long long tiles = ((p.inner + p.TI - 1) / p.TI) * ((p.outer + p.TO - 1) / p.TO);
        const size_t smem = sizeof(C) * ((size_t)2 * P * p.TO * p.TI + P);
        if (smem > 227 * 1024) throw Error(AIM_E_GRID, "FFT length exceeds the shared-memory tile capacity");
        ensure_smem_attr(fft_pp_kernel<C>);
        fft_pp_kernel<C><<<(unsigned)tiles, kFftThreads, smem, s>>>(p);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess)
            throw Error(AIM_E_CUDA, "fft_pp_kernel P=" + std::to_string(P) + " tiles=" + std::to_string(tiles) +
                                        " smem=" + std::to_string(smem) + ": " + cudaGetErrorString(e));
    }
}

bool try_launch_fft_pass_tab(const FftPass& p, cudaStream_t s) {
    if (p.outer <= 0 || p.inner <= 0) return true;
    const char* ce = getenv("AIM_FFT_NOCT");
    if (p.prec == 1 || p.TI > 0 || (ce && ce[0] == '1')) return false;
    const bool ok = try_ct_pass<double2, Ct210, 2>(p, s) || try_ct_pass<double2, Ct784, (AIM_CT784_NL > 2 ? 1 : 2)>(p, s);
    if (ok) note_launch("fft_pass");
    return ok;
}

void launch_fft_pass(const FftPass& p, cudaStream_t s) {
    if (p.outer <= 0 || p.inner <= 0) return;
    if (p.jin || p.jout) throw Error(AIM_E_GRID, "launch_fft_pass: table-addressed passes go through try_launch_fft_pass_tab");
    if (p.prec == 1) launch_fft_pass_t<float2>(p, s);
    else launch_fft_pass_t<double2>(p, s);
    note_launch("fft_pass");
}

// planar pass: one CTA holds a (Py x Nz) plane in place, one butterfly per thread per stage
bool planar_supported(int Py, int Nz, int min_radix) {
    const size_t smem = sizeof(double2) * ((size_t)2 * Py * Nz + Py);
    return Nz <= kPlanarMaxNz && (long long)Nz * Py / min_radix <= kPlanarThreads && smem <= 200 * 1024;
}

template <class C, class K>
static void launch_planar(K kern, const PlanarPass& p, int threads, cudaStream_t s) {
    const int Py = p.ay.P;
    const long long tiles = 4LL * p.Px * ((p.R + p.RC - 1) / p.RC);
    const size_t smem = sizeof(C) * ((size_t)2 * Py * p.Nz * p.RC + Py);
    ensure_smem_attr(kern);
    const long long grid = persistent_grid(kern, threads, smem, tiles);
    kern<<<(unsigned)grid, threads, smem, s>>>(p, (int)tiles);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        throw Error(AIM_E_CUDA, "planar_yz_kernel Py=" + std::to_string(Py) + " Nz=" + std::to_string(p.Nz) +
                                    " RC=" + std::to_string(p.RC) + " threads=" + std::to_string(threads) +
                                    " smem=" + std::to_string(smem) + ": " + cudaGetErrorString(e));
}

template <class C, int NZ, class F, int MINB>
static bool try_ct_planar(PlanarPass p, cudaStream_t s) {
    if (p.ay.P != F::P || p.Nz != NZ || p.PyH != F::P / 2 + 1) return false;
    p.RC = 1;
    const long long tiles = 4LL * p.Px * p.R;
    const size_t smem = sizeof(C) * ((size_t)3 * F::P * NZ);
    auto kern = planar_ct_kernel<NZ, F, MINB, C>;
    ensure_smem_attr(kern);
    const long long grid = persistent_grid(kern, F::T, smem, tiles);
    kern<<<(unsigned)grid, F::T, smem, s>>>(p, (int)tiles);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        throw Error(AIM_E_CUDA, "planar_ct_kernel Py=" + std::to_string(F::P) + ": " + cudaGetErrorString(e));
    return true;
}

// NW warps per CTA: at least one half-warp per z line; more warps so that the
// Toeplitz step (one thread per ky) runs in one round.
#ifndef AIM_PLANAR4_NW11
#define AIM_PLANAR4_NW11 6
#endif
template <int NZ, int N1, int N2, int NW>
static bool try_planar4(const PlanarPass& p, cudaStream_t s) {
    constexpr int Py = N1 * N2;
    if (p.ay.P != Py || p.Nz != NZ || p.PyH != Py / 2 + 1) return false;
    const long long tiles = 4LL * p.Px * p.R;
    const size_t smem = sizeof(double2) * ((size_t)2 * Py * NZ + (Py / 2 + 1) * NZ + Py);
    auto kern = planar4_kernel<NZ, N1, N2, NW>;
    constexpr int T = 32 * NW;
    ensure_smem_attr(kern);
    const long long grid = persistent_grid(kern, T, smem, tiles);
    kern<<<(unsigned)grid, T, smem, s>>>(p, (int)tiles);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw Error(AIM_E_CUDA, std::string("planar4_kernel: ") + cudaGetErrorString(e));
    return true;
}

template <class C>
static void launch_planar_yz_t(PlanarPass p, cudaStream_t s) {
    if constexpr (sizeof(C) == 16) {
        // four-step register kernel (AIM_PLANAR_KERNEL=stockham forces the stage kernel, A/B timing only)
        const char* e = getenv("AIM_PLANAR_KERNEL");
        if (!(e && !strcmp(e, "stockham")) && (try_planar4<11, 14, 15, AIM_PLANAR4_NW11>(p, s) || try_planar4<7, 4, 6, 4>(p, s)))
            return;
    }
    if (try_ct_planar<C, 11, Ct210z11, 2>(p, s) || try_ct_planar<C, 7, Ct24z7, 2>(p, s)) return;
    const int Py = p.ay.P;
    const int rc_fft = (int)(kPlanarThreads * (long long)p.ay.min_radix / ((long long)Py * p.Nz));
    p.RC = std::max(1, std::min({p.R, rc_fft, kPlanarThreads / p.Nz}));
    while (p.RC > 1 && sizeof(C) * ((size_t)2 * Py * p.Nz * p.RC + Py) > 110 * 1024) --p.RC;
    // one butterfly per thread per FFT stage; one (ky, rhs) z line per thread in the convolution
    const int bfly = (int)((long long)p.Nz * p.RC * Py / p.ay.min_radix);
    const int threads = std::min(kPlanarThreads, 32 * ((std::max({bfly, Py * p.RC, p.Nz * p.RC}) + 31) / 32));
    switch (p.Nz) {
#define PZ(NZ) case NZ: launch_planar<C>(planar_yz_kernel<NZ, RtPlan, kPlanarThreads, 2, C>, p, threads, s); break;
        PZ(1) PZ(2) PZ(3) PZ(4) PZ(5) PZ(6) PZ(7) PZ(8) PZ(9) PZ(10) PZ(11) PZ(12) PZ(13) PZ(14) PZ(15) PZ(16)
#undef PZ
        default: throw Error(AIM_E_GRID, "planar pass: Nz out of range");
    }
}

void launch_planar_yz(const PlanarPass& p, cudaStream_t s) {
    if (p.prec == 1) launch_planar_yz_t<float2>(p, s);
    else launch_planar_yz_t<double2>(p, s);
    note_launch("planar_yz");
}

}  // namespace aim
