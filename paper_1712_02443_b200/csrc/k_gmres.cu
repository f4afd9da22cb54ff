// Restarted GMRES on the device (PAPER.md:510-511
// "we solve the linear system ... iteratively using the generalized minimal
// residual (GMRES) algorithm"; reading D15).
//
// Krylov basis V [restart+1][N] and all vector work stay in HBM; the host
// keeps only the (restart+1) x restart Hessenberg matrix and the Givens
// rotations.  Arnoldi uses classical Gram-Schmidt applied twice (CGS2):
// each pass is one fused multi-dot kernel (partials per block, fixed-order
// second stage => deterministic) and one fused multi-axpy kernel.
#include <math.h>

#include <algorithm>
#include <complex>
#include <functional>
#include <vector>

#include "aim_internal.cuh"

namespace aim {

using cplx = std::complex<double>;

static constexpr int kDotBlocks = 296;  // 2 x 148 SMs
static constexpr int kDotThreads = 256;
static constexpr int kMaxBasis = 1024;

__constant__ double2 c_coef[kMaxBasis];

// partial[b][i] = sum_{e in block b's range} conj(V_i[e]) w[e], i < nv
__global__ void __launch_bounds__(kDotThreads) multidot_kernel(const double2* __restrict__ V, long long N, int nv,
                                                               const double2* __restrict__ w,
                                                               double2* __restrict__ partial) {
    __shared__ double2 red[kDotThreads / 32];
    const long long chunk = (N + gridDim.x - 1) / gridDim.x;
    const long long a = blockIdx.x * chunk, b = min(N, a + chunk);
    const int lane = threadIdx.x & 31, warp = threadIdx.x / 32;
    for (int i = 0; i < nv; ++i) {
        const double2* Vi = V + (long long)i * N;
        double2 s = make_double2(0, 0);
        for (long long e = a + threadIdx.x; e < b; e += blockDim.x) {
            const double2 v = Vi[e], x = w[e];
            s.x += v.x * x.x + v.y * x.y;
            s.y += v.x * x.y - v.y * x.x;
        }
        for (int off = 16; off; off >>= 1) {
            s.x += __shfl_xor_sync(0xffffffffu, s.x, off);
            s.y += __shfl_xor_sync(0xffffffffu, s.y, off);
        }
        if (lane == 0) red[warp] = s;
        __syncthreads();
        if (threadIdx.x == 0) {
            double2 t = make_double2(0, 0);
            for (int q = 0; q < kDotThreads / 32; ++q) { t.x += red[q].x; t.y += red[q].y; }
            partial[(long long)blockIdx.x * nv + i] = t;
        }
        __syncthreads();
    }
}

// out[i] = sum_b partial[b][i] in block order
__global__ void multidot_final(const double2* __restrict__ partial, int nb, int nv, double2* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nv) return;
    double2 t = make_double2(0, 0);
    for (int b = 0; b < nb; ++b) { t.x += partial[(long long)b * nv + i].x; t.y += partial[(long long)b * nv + i].y; }
    out[i] = t;
}

// w[e] += sign * sum_i coef[i] V_i[e]
__global__ void multiaxpy_kernel(const double2* __restrict__ V, long long N, int nv, double sign,
                                 double2* __restrict__ w) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= N) return;
    double2 acc = w[e];
    for (int i = 0; i < nv; ++i) {
        const double2 c = c_coef[i], v = V[(long long)i * N + e];
        acc.x += sign * (c.x * v.x - c.y * v.y);
        acc.y += sign * (c.x * v.y + c.y * v.x);
    }
    w[e] = acc;
}

__global__ void scale_copy_kernel(const double2* __restrict__ a, long long N, double s, double2* __restrict__ b) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < N) b[e] = make_double2(a[e].x * s, a[e].y * s);
}

// r = b - Ax
__global__ void residual_kernel(const double2* __restrict__ b, const double2* __restrict__ Ax, long long N,
                                double2* __restrict__ r) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < N) r[e] = make_double2(b[e].x - Ax[e].x, b[e].y - Ax[e].y);
}

struct Gm {
    aim_plan* p;
    cudaStream_t s;
    double2* part;
    double2* dres;
    std::vector<double2> hbuf;

    void dots(const double2* V, int nv, const double2* w, cplx* out) {
        multidot_kernel<<<kDotBlocks, kDotThreads, 0, s>>>(V, p->N, nv, w, part);
        note_launch("gmres_multidot");
        multidot_final<<<(nv + 127) / 128, 128, 0, s>>>(part, kDotBlocks, nv, dres);
        note_launch("gmres_multidot_final");
        hbuf.resize(nv);
        AIM_CUDA(cudaMemcpyAsync(hbuf.data(), dres, sizeof(double2) * nv, cudaMemcpyDeviceToHost, s));
        AIM_CUDA(cudaStreamSynchronize(s));
        for (int i = 0; i < nv; ++i) out[i] = cplx(hbuf[i].x, hbuf[i].y);
    }
    double norm(const double2* w) {
        cplx d;
        dots(w, 1, w, &d);
        return sqrt(std::max(0.0, d.real()));
    }
    void axpy(const double2* V, int nv, const cplx* c, double sign, double2* w) {
        std::vector<double2> h(nv);
        for (int i = 0; i < nv; ++i) h[i] = make_double2(c[i].real(), c[i].imag());
        AIM_CUDA(cudaMemcpyToSymbolAsync(c_coef, h.data(), sizeof(double2) * nv, 0, cudaMemcpyHostToDevice, s));
        multiaxpy_kernel<<<(unsigned)((p->N + 255) / 256), 256, 0, s>>>(V, p->N, nv, sign, w);
        note_launch("gmres_multiaxpy");
    }
    void scale(const double2* a, double f, double2* b) {
        scale_copy_kernel<<<(unsigned)((p->N + 255) / 256), 256, 0, s>>>(a, p->N, f, b);
        note_launch("gmres_scale");
    }
};

int gmres(aim_plan* p, const double2* b, double2* x, int restart, double tol, int max_iters, int fixed_iters,
          int* iters_out, double* rel_out) {
    return gmres_with(p, [p](const double2* in, double2* out, cudaStream_t st) { matvec(p, in, out, 1, st); }, b, x,
                      restart, tol, max_iters, fixed_iters, iters_out, rel_out);
}

// The solver with any operator: `p` holds the workspace (and N, the stream),
// `mv` applies the operator (single plan, or the slab-decomposed product with
// replicated vectors -- every rank then runs the identical iteration).
int gmres_with(aim_plan* p, const std::function<void(const double2*, double2*, cudaStream_t)>& mv,
               const double2* b, double2* x, int restart, double tol, int max_iters, int fixed_iters,
               int* iters_out, double* rel_out) {
    if (restart < 1 || restart + 1 > kMaxBasis) throw Error(AIM_E_ARG, "restart must be in [1, 1023]");
    if (max_iters <= 0) max_iters = 20000;
    const long long N = p->N;
    cudaStream_t s = p->stream;
    if (p->gm_restart < restart) {
        p->release(p->gm_V);
        p->release(p->gm_w);
        p->release(p->gm_part);
        p->gm_V = p->alloc<double2>((size_t)(restart + 1) * N);
        p->gm_w = p->alloc<double2>(N);
        p->gm_part = p->alloc<double2>((size_t)kDotBlocks * (restart + 1) + kMaxBasis);
        p->gm_restart = restart;
    }
    Gm g{p, s, p->gm_part, p->gm_part + (size_t)kDotBlocks * (restart + 1), {}};
    double2* V = p->gm_V;
    double2* w = p->gm_w;
    const int limit = fixed_iters > 0 ? fixed_iters : max_iters;

    AIM_CUDA(cudaMemsetAsync(x, 0, sizeof(double2) * N, s));
    const double bnorm = g.norm(b);
    if (bnorm == 0.0) {
        AIM_CUDA(cudaStreamSynchronize(s));
        if (iters_out) *iters_out = 0;
        if (rel_out) *rel_out = 0.0;
        return AIM_OK;
    }
    // r0 = b (x0 = 0)
    double beta = bnorm;
    g.scale(b, 1.0 / beta, V);
    int total = 0;
    double rel = 1.0;
    std::vector<cplx> H((size_t)(restart + 1) * restart), gv(restart + 1), sn(restart), h1(restart + 1),
        h2(restart + 1);
    std::vector<double> cs(restart);
    auto Hij = [&](int i, int j) -> cplx& { return H[(size_t)i * restart + j]; };
    while (true) {
        std::fill(H.begin(), H.end(), cplx(0));
        std::fill(gv.begin(), gv.end(), cplx(0));
        gv[0] = beta;
        int jd = 0;
        bool stop = false;
        for (int j = 0; j < restart; ++j) {
            mv(V + (size_t)j * N, w, s);
            // CGS2: two classical Gram-Schmidt passes
            g.dots(V, j + 1, w, h1.data());
            g.axpy(V, j + 1, h1.data(), -1.0, w);
            g.dots(V, j + 1, w, h2.data());
            g.axpy(V, j + 1, h2.data(), -1.0, w);
            for (int i = 0; i <= j; ++i) Hij(i, j) = h1[i] + h2[i];
            const double hn = g.norm(w);
            Hij(j + 1, j) = hn;
            if (hn > 0) g.scale(w, 1.0 / hn, V + (size_t)(j + 1) * N);
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
            if (total >= limit) { stop = true; break; }
            if (fixed_iters <= 0 && est <= tol) break;
            if (hn == 0) break;
        }
        // y = H^-1 g (upper triangular), x += V y
        std::vector<cplx> yv(jd);
        for (int i = jd - 1; i >= 0; --i) {
            cplx t = gv[i];
            for (int q = i + 1; q < jd; ++q) t -= Hij(i, q) * yv[q];
            yv[i] = t / Hij(i, i);
        }
        if (jd) g.axpy(V, jd, yv.data(), +1.0, x);
        // true residual r = b - A x into V[0]
        mv(x, w, s);
        residual_kernel<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(b, w, N, V);
        note_launch("gmres_residual");
        beta = g.norm(V);
        rel = beta / bnorm;
        if (stop || (fixed_iters <= 0 && rel <= tol) || beta == 0.0) break;
        g.scale(V, 1.0 / beta, V);
    }
    AIM_CUDA(cudaStreamSynchronize(s));
    if (iters_out) *iters_out = total;
    if (rel_out) *rel_out = rel;
    return rel <= tol ? AIM_OK : AIM_NOT_CONVERGED;
}

}  // namespace aim
