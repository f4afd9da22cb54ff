// Fused y/z convolution pass for thin planar grids (conv mode 2: C3, C4),
// included by k_fft.cu (shares its register radices and twiddle constants).
//
// Step (ii) of the AIM matvec (eq. AIM_step2) on the
// x-transformed grid W1[4][Px][Ny][Nz] (one right-hand side): for every
// (component, kx) plane -- one CTA, the whole [Py][Nz] plane in shared memory:
//   1. TMA bulk copy of the plane's Ny x Nz values (contiguous), zero rows
//      Ny .. Py-1 (the y zero padding, D11);
//   2. forward y FFT of length Py = R1 R2 R3 in place: decimation in
//      frequency, three radix stages in registers, output in digit-reversed
//      order (position k1 S1 + k2 R3 + k3 holds ky = k1 + R1 k2 + R1 R2 k3);
//   3. z convolution as the symmetric Toeplitz product with the 2-D spectrum
//      G2(kx, ky, |dz|) (1/(Px Py) folded in), thread per ky line;
//   4. inverse y FFT in place (decimation in time, digit-reversed -> natural);
//   5. TMA bulk store of rows 0 .. Ny-1 (the pruning).
// One HBM round trip of the plane instead of the three passes (y forward to
// the y-padded W2, z Toeplitz on W2, y inverse back) of the unfused mode 2.

#ifndef AIM_YM2_PRUNE
#define AIM_YM2_PRUNE 0   // 1: skip the zero-padding rows in the first forward / last inverse stage (parity-green,
                          // measured neutral on C4: 0.635 vs 0.638 ms at equal clocks, so off by default)
#endif

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* m, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* m, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(m)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, unsigned phase) {
    asm volatile(
        "{\n .reg .pred P;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra WAIT_%=;\n}\n" ::"r"(
            smem_u32(m)),
        "r"(phase)
        : "memory");
}
// global -> shared bulk copy (TMA, no tensor map), completion on the mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* m) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(m))
                 : "memory");
}
// shared -> global bulk copy (TMA), bulk-group completion
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// One in-place radix-R stage over the tile [P][NZ]: butterfly j (block j / ST,
// offset m = j % ST) on positions base + t ST, base = (j / ST) R ST + m.
//   DIF (forward): b = DFT_R(a) (sign -), b_k *= w_{R ST}^{m k}
//   DIT (inverse): a_t *= conj(w_{R ST}^{m t}), b = DFT_R(a) (sign +)
// TLD < R: only inputs t < TLD are read, the others are zero (first forward
// stage: rows >= P/2 are y padding); TST < R: only outputs t < TST are stored
// (last inverse stage: rows >= P/2 are pruned), the rest of the butterfly's
// outputs is dead code.
template <int P, int R, int ST, int NZ, bool DIF, int TLD = R, int TST = R>
__device__ __forceinline__ void ym2_stage(double2* tile, const double2* tw) {
    if constexpr (R == 1) return;        // two-stage plans (R3 = 1)
    constexpr int NB = P / R;            // butterflies per column
    constexpr int TWS = P / (R * ST);    // twiddle exponent scale
#pragma unroll 1
    for (int q = threadIdx.x; q < NB * NZ; q += blockDim.x) {
        const int j = q / NZ, l = q - (q / NZ) * NZ;
        const int m = j % ST;
        const int base = (j / ST) * R * ST + m;
        double2 a[R];
#pragma unroll
        for (int t = 0; t < R; ++t) a[t] = t < TLD ? tile[(base + t * ST) * NZ + l] : make_double2(0, 0);
        if constexpr (DIF) {
            dft<R>(a, -1.0);
#pragma unroll
            for (int k = 1; k < R; ++k) {
                const int e = (m * k * TWS) % P;
                if (e) a[k] = cmul(a[k], tw[e]);
            }
        } else {
#pragma unroll
            for (int t = 1; t < R; ++t) {
                const int e = (m * t * TWS) % P;
                if (e) {
                    const double2 w = tw[e];
                    a[t] = cmul(a[t], make_double2(w.x, -w.y));
                }
            }
            dft<R>(a, 1.0);
        }
#pragma unroll
        for (int t = 0; t < R; ++t)
            if (t < TST) tile[(base + t * ST) * NZ + l] = a[t];
    }
}

template <int P, int R1, int R2, int R3, int NZ, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) ymode2_kernel(double2* __restrict__ W, int Ny, int Px, int PyH,
                                                           const double2* __restrict__ spec,
                                                           const double2* __restrict__ twg, int planes) {
    static_assert(R1 * R2 * R3 == P, "radices");
    constexpr int S1 = R2 * R3;
    // rows >= P/2 are zero padding on input and pruned on output (Ny <= (P + 1) / 2):
    // the first forward stage reads, and the last inverse stage writes, only t < TH
    constexpr int TH = AIM_YM2_PRUNE ? (R1 + 1) / 2 : R1;
    constexpr int ZEND = (TH * S1 < P ? TH * S1 : P) * NZ;
    extern __shared__ __align__(128) unsigned char ym2_raw[];
    double2* tile = reinterpret_cast<double2*>(ym2_raw);     // [P][NZ]
    double2* tw = tile + P * NZ;                             // [P]
    __shared__ __align__(8) uint64_t mbar;
    for (int e = threadIdx.x; e < P; e += blockDim.x) tw[e] = twg[e];
    if (threadIdx.x == 0) {
        mbar_init(&mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    const unsigned bytes = (unsigned)(Ny * NZ * sizeof(double2));
    unsigned phase = 0;
    for (int q = blockIdx.x; q < planes; q += gridDim.x) {
        double2* plane = W + (long long)q * Ny * NZ;
        const int kx = q % Px;
        const int ax = min(kx, Px - kx);
        // 1. load (the previous plane's store must have read the tile)
        fence_async_smem();
        __syncthreads();
        if (threadIdx.x == 0) {
            bulk_wait_read();
            mbar_expect_tx(&mbar, bytes);
            bulk_g2s(tile, plane, bytes, &mbar);
        }
        for (int e = Ny * NZ + threadIdx.x; e < ZEND; e += blockDim.x) tile[e] = make_double2(0, 0);
        mbar_wait(&mbar, phase);
        phase ^= 1;
        // the next plane of this CTA into L2 while this one is transformed
        if (threadIdx.x == 0 && q + gridDim.x < planes)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(W + (long long)(q + gridDim.x) * Ny * NZ),
                         "r"(bytes)
                         : "memory");
        __syncthreads();
        // 2. forward y FFT (DIF), digit-reversed output
        ym2_stage<P, R1, S1, NZ, true, TH, R1>(tile, tw);
        __syncthreads();
        ym2_stage<P, R2, R3, NZ, true>(tile, tw);
        __syncthreads();
        ym2_stage<P, R3, 1, NZ, true>(tile, tw);
        __syncthreads();
        // 3. z Toeplitz with G2(kx, ky, |dz|)
        const double2* g2 = spec + (long long)ax * PyH * NZ;
#pragma unroll 1
        for (int p = threadIdx.x; p < P; p += blockDim.x) {
            const int k1 = p / S1, k2 = (p / R3) % R2, k3 = p % R3;
            const int ky = k1 + R1 * k2 + R1 * R2 * k3;
            const int ay = min(ky, P - ky);
            const double2* g = g2 + ay * NZ;
            double2* row = tile + p * NZ;
            double2 gk[NZ], in[NZ];
#pragma unroll
            for (int d = 0; d < NZ; ++d) gk[d] = __ldg(&g[d]);
#pragma unroll
            for (int z = 0; z < NZ; ++z) in[z] = row[z];
#pragma unroll
            for (int z = 0; z < NZ; ++z) {
                double2 acc = cmul(gk[0], in[z]);
#pragma unroll
                for (int d = 1; d < NZ; ++d) {
                    if (z - d < 0 && z + d >= NZ) continue;
                    double2 sum = z - d >= 0 ? in[z - d] : make_double2(0, 0);
                    if (z + d < NZ) sum = z - d >= 0 ? cadd(sum, in[z + d]) : in[z + d];
                    acc.x = fma(gk[d].x, sum.x, fma(-gk[d].y, sum.y, acc.x));
                    acc.y = fma(gk[d].x, sum.y, fma(gk[d].y, sum.x, acc.y));
                }
                row[z] = acc;
            }
        }
        __syncthreads();
        // 4. inverse y FFT (DIT), natural output
        ym2_stage<P, R3, 1, NZ, false>(tile, tw);
        __syncthreads();
        ym2_stage<P, R2, R3, NZ, false>(tile, tw);
        __syncthreads();
        ym2_stage<P, R1, S1, NZ, false, R1, TH>(tile, tw);
        // 5. store rows 0 .. Ny-1
        fence_async_smem();
        __syncthreads();
        if (threadIdx.x == 0) bulk_s2g(plane, tile, bytes);
    }
    if (threadIdx.x == 0) bulk_wait_all();
}

// ---------------------------------------------------- 2-CTA cluster version
// The same pass with each plane split over a cluster of two CTAs (two SMs):
// CTA q holds z columns [q NH, q NH + n_q) of the plane (NH = ceil(Nz/2)),
// loaded and stored with one TMA bulk copy per row, and runs the y FFTs on
// them; the z Toeplitz of ky line p needs all Nz values, so the peer's
// columns are read from its shared memory (DSMEM, ld.shared::cluster), one
// cluster barrier per round of lines separating the reads from the in-place
// writes.  Half the shared memory per CTA (C4: 88 KB) -> two CTAs per SM.
__device__ __forceinline__ unsigned cl_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned cl_id() {
    unsigned r;
    asm volatile("mov.u32 %0, %%clusterid.x;\n" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned cl_count() {
    unsigned r;
    asm volatile("mov.u32 %0, %%nclusterid.x;\n" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cl_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ unsigned cl_map(const void* p, unsigned rank) {
    unsigned a;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(a) : "r"(smem_u32(p)), "r"(rank));
    return a;
}
__device__ __forceinline__ double2 ld_dsmem(unsigned addr) {
    double2 v;
    asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(addr) : "memory");
    return v;
}

// radix-R stage over the first nq of NH columns (row stride NH)
template <int P, int R, int ST, int NH, bool DIF>
__device__ __forceinline__ void ym2c_stage(double2* tile, const double2* tw, int nq) {
    constexpr int NB = P / R;
    constexpr int TWS = P / (R * ST);
#pragma unroll 1
    for (int q = threadIdx.x; q < NB * nq; q += blockDim.x) {
        const int j = q / nq, l = q - (q / nq) * nq;
        const int m = j % ST;
        const int base = (j / ST) * R * ST + m;
        double2 a[R];
#pragma unroll
        for (int t = 0; t < R; ++t) a[t] = tile[(base + t * ST) * NH + l];
        if constexpr (DIF) {
            dft<R>(a, -1.0);
#pragma unroll
            for (int k = 1; k < R; ++k) {
                const int e = (m * k * TWS) % P;
                if (e) a[k] = cmul(a[k], tw[e]);
            }
        } else {
#pragma unroll
            for (int t = 1; t < R; ++t) {
                const int e = (m * t * TWS) % P;
                if (e) {
                    const double2 w = tw[e];
                    a[t] = cmul(a[t], make_double2(w.x, -w.y));
                }
            }
            dft<R>(a, 1.0);
        }
#pragma unroll
        for (int t = 0; t < R; ++t) tile[(base + t * ST) * NH + l] = a[t];
    }
}

// z Toeplitz of ky line p for the columns of cluster rank Q (compile-time
// column ranges, so the line stays in registers): out[j] = sum_z' G2(|z - z'|)
// in[z'], z = Q NH + j; the peer's columns come from its shared memory.
template <int NZ, int Q>
__device__ __forceinline__ void ym2c_toeplitz(const double2* tile, unsigned peer, int p, const double2* g,
                                              double2* out) {
    constexpr int NH = (NZ + 1) / 2;
    constexpr int z0 = Q * NH, nq = Q ? NZ - NH : NH;
    constexpr int z0p = Q ? 0 : NH, nqp = Q ? NH : NZ - NH;
    double2 in[NZ];
#pragma unroll
    for (int z = 0; z < NZ; ++z) {
        if (z >= z0 && z < z0 + nq) in[z] = tile[p * NH + z - z0];
        else if (z >= z0p && z < z0p + nqp) in[z] = ld_dsmem(peer + (unsigned)((p * NH + z - z0p) * 16));
        else in[z] = make_double2(0, 0);
    }
#pragma unroll
    for (int j = 0; j < NH; ++j) out[j] = make_double2(0, 0);
#pragma unroll
    for (int d = 0; d < NZ; ++d) {
        const double2 gd = __ldg(&g[d]);
#pragma unroll
        for (int j = 0; j < nq; ++j) {
            const int z = z0 + j;
            if (z - d < 0 && (d == 0 || z + d >= NZ)) continue;
            double2 sum = z - d >= 0 ? in[z - d] : make_double2(0, 0);
            if (d && z + d < NZ) sum = z - d >= 0 ? cadd(sum, in[z + d]) : in[z + d];
            out[j].x = fma(gd.x, sum.x, fma(-gd.y, sum.y, out[j].x));
            out[j].y = fma(gd.x, sum.y, fma(gd.y, sum.x, out[j].y));
        }
    }
}

template <int P, int R1, int R2, int R3, int NZ, int NT>
__global__ void __launch_bounds__(NT, 2) ymode2c_kernel(double2* __restrict__ W, int Ny, int Px, int PyH,
                                                        const double2* __restrict__ spec,
                                                        const double2* __restrict__ twg, int planes) {
    constexpr int NH = (NZ + 1) / 2, S1 = R2 * R3;
    extern __shared__ __align__(128) unsigned char ym2c_raw[];
    double2* tile = reinterpret_cast<double2*>(ym2c_raw);    // [P][NH]
    double2* tw = tile + P * NH;                             // [P]
    __shared__ __align__(8) uint64_t mbar;
    const unsigned q = cl_rank();
    const int z0 = (int)q * NH, nq = q ? NZ - NH : NH;
    const int z0p = q ? 0 : NH, nqp = q ? NH : NZ - NH;       // the peer's columns
    for (int e = threadIdx.x; e < P; e += blockDim.x) tw[e] = twg[e];
    if (threadIdx.x == 0) {
        mbar_init(&mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    cl_sync();
    const unsigned peer = cl_map(tile, q ^ 1u);
    unsigned phase = 0;
    for (int pl = (int)cl_id(); pl < planes; pl += (int)cl_count()) {
        double2* plane = W + (long long)pl * Ny * NZ;
        const int kx = pl % Px;
        const int ax = min(kx, Px - kx);
        // 1. load my columns of rows 0 .. Ny-1 (one bulk copy per row), zero the y padding
        fence_async_smem();
        bulk_wait_read();            // my previous bulk stores have read the tile
        __syncthreads();
        if (threadIdx.x == 0) mbar_expect_tx(&mbar, (unsigned)(Ny * nq * sizeof(double2)));
        __syncthreads();
        for (int row = threadIdx.x; row < Ny; row += NT)
            bulk_g2s(tile + row * NH, plane + (long long)row * NZ + z0, (unsigned)(nq * sizeof(double2)), &mbar);
        for (int e = Ny * NH + threadIdx.x; e < P * NH; e += NT) tile[e] = make_double2(0, 0);
        mbar_wait(&mbar, phase);
        phase ^= 1;
        __syncthreads();
        // 2. forward y FFT on my columns
        ym2c_stage<P, R1, S1, NH, true>(tile, tw, nq);
        __syncthreads();
        ym2c_stage<P, R2, R3, NH, true>(tile, tw, nq);
        __syncthreads();
        ym2c_stage<P, R3, 1, NH, true>(tile, tw, nq);
        __syncthreads();
        cl_sync();                   // the peer's forward transform is complete
        // 3. z Toeplitz for my columns, rounds of NT lines
        const double2* g2 = spec + (long long)ax * PyH * NZ;
#pragma unroll 1
        for (int p0 = 0; p0 < P; p0 += NT) {
            const int p = p0 + threadIdx.x;
            double2 out[NH];
            if (p < P) {
                const int k1 = p / S1, k2 = (p / R3) % R2, k3 = p % R3;
                const int ky = k1 + R1 * k2 + R1 * R2 * k3;
                const int ay = min(ky, P - ky);
                const double2* g = g2 + ay * NZ;
                if (q == 0) ym2c_toeplitz<NZ, 0>(tile, peer, p, g, out);
                else ym2c_toeplitz<NZ, 1>(tile, peer, p, g, out);
            }
            cl_sync();               // every read of this round's lines (both CTAs) is done
            if (p < P)
#pragma unroll
                for (int j = 0; j < NH; ++j)
                    if (j < nq) tile[p * NH + j] = out[j];
        }
        __syncthreads();
        // 4. inverse y FFT on my columns
        ym2c_stage<P, R3, 1, NH, false>(tile, tw, nq);
        __syncthreads();
        ym2c_stage<P, R2, R3, NH, false>(tile, tw, nq);
        __syncthreads();
        ym2c_stage<P, R1, S1, NH, false>(tile, tw, nq);
        // 5. store rows 0 .. Ny-1 of my columns
        fence_async_smem();
        __syncthreads();
        for (int row = threadIdx.x; row < Ny; row += NT)
            bulk_s2g(plane + (long long)row * NZ + z0, tile + row * NH, (unsigned)(nq * sizeof(double2)));
    }
    bulk_wait_all();
    cl_sync();                       // no CTA leaves while its peer may read its shared memory
}

// Fused mode-2 pass for the compiled plans (Py, Nz) = (784, 14) (C4) and
// (486, 13) (C3); complex128, one right-hand side.  Returns false if no plan
// matches (the caller runs the three separate passes).  AIM_YZ_FUSED=0
// disables it (A/B and parity tests).
bool launch_ymode2(void* W, int prec, int Px, int Ny, int Nz, int Py, int R, const void* spec, const FftAxis& ay,
                   cudaStream_t s) {
    const char* env = getenv("AIM_YZ_FUSED");
    const bool off = env && env[0] == '0';
    if (off || prec != 0 || R != 1) return false;
    if (2 * Ny > Py + 1) return false;   // the pruned first/last stages assume rows >= ceil(Py/2) are padding
    int dev = 0;
    AIM_CUDA(cudaGetDevice(&dev));
    const int planes = 4 * Px;
    const int PyH = Py / 2 + 1;
    // the 2-CTA cluster variant is opt-in: measured slower on C4 (1.19 vs 0.63 ms)
    // and C3 (0.35 vs 0.21 ms) -- 386 row bulk copies per CTA, DSMEM line reads
    // and four cluster barriers per plane cost more than the doubled occupancy gains
    const char* envc = getenv("AIM_YZ_CLUSTER");
    const bool cluster = envc && envc[0] == '1';
#define YM2C_CASE(PP, A, B, C, NZ, NT)                                                                        \
    if (cluster && Py == PP && Nz == NZ) {                                                                    \
        const size_t smem = sizeof(double2) * (size_t)PP * ((NZ + 1) / 2 + 1);                               \
        static unsigned long long mask = 0; /* cudaFuncSetAttribute is per device */                         \
        if (!(mask >> (dev & 63) & 1ULL)) {                                                                   \
            AIM_CUDA(cudaFuncSetAttribute(ymode2c_kernel<PP, A, B, C, NZ, NT>,                                \
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));            \
            mask |= 1ULL << (dev & 63);                                                                       \
        }                                                                                                     \
        cudaLaunchConfig_t cfg = {};                                                                          \
        cfg.gridDim = dim3(2 * 148, 1, 1);                                                                    \
        cfg.blockDim = dim3(NT, 1, 1);                                                                        \
        cfg.dynamicSmemBytes = smem;                                                                          \
        cfg.stream = s;                                                                                       \
        cudaLaunchAttribute at[1];                                                                            \
        at[0].id = cudaLaunchAttributeClusterDimension;                                                       \
        at[0].val.clusterDim.x = 2;                                                                           \
        at[0].val.clusterDim.y = 1;                                                                           \
        at[0].val.clusterDim.z = 1;                                                                           \
        cfg.attrs = at;                                                                                       \
        cfg.numAttrs = 1;                                                                                     \
        AIM_CUDA(cudaLaunchKernelEx(&cfg, ymode2c_kernel<PP, A, B, C, NZ, NT>, (double2*)W, Ny, Px, PyH,      \
                                    (const double2*)spec, (const double2*)ay.tw, planes));                    \
        note_launch("ymode2c");                                                                               \
        return true;                                                                                          \
    }
    YM2C_CASE(784, 16, 7, 7, 14, 256)
    YM2C_CASE(486, 9, 9, 6, 13, 256)
#undef YM2C_CASE
#define YM2_CASE(PP, A, B, C, NZ, NT, MINB)                                                                   \
    if (Py == PP && Nz == NZ) {                                                                               \
        const size_t smem = sizeof(double2) * (size_t)PP * (NZ + 1);                                          \
        static unsigned long long mask = 0; /* cudaFuncSetAttribute is per device */                         \
        if (!(mask >> (dev & 63) & 1ULL)) {                                                                   \
            AIM_CUDA(cudaFuncSetAttribute(ymode2_kernel<PP, A, B, C, NZ, NT, MINB>,                           \
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));            \
            if (smem_carveout_max())                                                                          \
                AIM_CUDA(cudaFuncSetAttribute(ymode2_kernel<PP, A, B, C, NZ, NT, MINB>,                       \
                                              cudaFuncAttributePreferredSharedMemoryCarveout, 100));          \
            mask |= 1ULL << (dev & 63);                                                                       \
        }                                                                                                     \
        ymode2_kernel<PP, A, B, C, NZ, NT, MINB><<<148 * MINB, NT, smem, s>>>(                                \
            (double2*)W, Ny, Px, PyH, (const double2*)spec, ay.tw, planes);                                   \
        note_launch("ymode2");                                                                                \
        return true;                                                                                          \
    }
    // C4: 784 = 28 x 28 in two in-place stages (one 28-point butterfly per
    // thread and column per stage, 392 threads) unless AIM_YM2_PLAN=3 selects
    // the three-stage 16 x 7 x 7 plan
    const char* envp = getenv("AIM_YM2_PLAN");
    const bool three = envp && envp[0] == '3';
    if (!three) YM2_CASE(784, 28, 28, 1, 14, 392, 1)
    YM2_CASE(784, 16, 7, 7, 14, 448, 1)
    YM2_CASE(486, 9, 9, 6, 13, 256, 2)
#undef YM2_CASE
    return false;
}
