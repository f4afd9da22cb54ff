// C ABI of the AIM library (include/aim.h) and the host part of plan
// construction (setup steps S0-S1 of SURVEY.md §8(a)):
//   S0 RWG geometry and the 7-point Radon/Dunavant rule (D7)
//      on every triangle;
//   S1 stencil bases s_n = floor(c_n/h - (M-1)/2 + 1e-7) (D3), grid box (D4)
//      and 7-smooth FFT sizes P_a >= 2 N_a - 1 (D11).
// Device-side setup (S2-S4) is in k_plan.cu; the per-matvec kernels are in
// k_matvec.cu / k_fft.cu and GMRES in k_gmres.cu.
#include <math.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <climits>
#include <cstring>
#include <string>
#include <vector>

#include "aim_internal.cuh"

namespace aim {

static thread_local std::string g_err;
static thread_local long long g_launches = 0;

std::string& last_error() { return g_err; }
long long launch_counter() { return g_launches; }
void add_launches(long long n) { g_launches += n; }

void note_launch(const char* name) {
    ++g_launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw Error(AIM_E_CUDA, std::string("launch ") + name + ": " + cudaGetErrorString(e));
    // AIM_SYNC_DEBUG=1: synchronise after every launch so a fault names its kernel
    static const bool sync_debug = getenv("AIM_SYNC_DEBUG") && getenv("AIM_SYNC_DEBUG")[0] == '1';
    if (sync_debug) {
        e = cudaDeviceSynchronize();
        if (e != cudaSuccess) throw Error(AIM_E_CUDA, std::string("kernel ") + name + ": " + cudaGetErrorString(e));
    }
}

// 7-point degree-5 rule (Radon; Dunavant's 7-point rule), D7
static void dunavant7(double bary[7][3], double w[7]) {
    const double s15 = sqrt(15.0);
    const double a1 = (6.0 - s15) / 21.0, a2 = (6.0 + s15) / 21.0;
    const double w1 = (155.0 - s15) / 1200.0, w2 = (155.0 + s15) / 1200.0;
    bary[0][0] = bary[0][1] = bary[0][2] = 1.0 / 3.0;
    w[0] = 9.0 / 40.0;
    const double as[2] = {a1, a2}, ws[2] = {w1, w2};
    for (int g = 0; g < 2; ++g) {
        const double a = as[g], b = 1.0 - 2.0 * a;
        for (int q = 0; q < 3; ++q) {
            for (int c = 0; c < 3; ++c) bary[1 + 3 * g + q][c] = (c == q) ? b : a;
            w[1 + 3 * g + q] = ws[g];
        }
    }
}

template <class T>
static T* upload(aim_plan* p, const std::vector<T>& h) {
    T* d = p->alloc<T>(h.size());
    h2d(d, h.data(), sizeof(T) * h.size(), p->stream);
    return d;
}

// complex64 plans (reading D16): round an fp64 table once at plan creation
__global__ void round_f32_kernel(const double* __restrict__ a, long long n, float* __restrict__ b) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        b[i] = (float)a[i];
}

static float* rounded_copy(aim_plan* p, const double* a, long long n, cudaStream_t s) {
    float* b = p->alloc<float>(n + 4);  // + bulk-copy slack (k_near_stream.cu)
    round_f32_kernel<<<(unsigned)std::min<long long>((n + 255) / 256, 148 * 16), 256, 0, s>>>(a, n, b);
    note_launch("round_f32");
    return b;
}

void make_c64_tables(aim_plan* p, cudaStream_t s) {
    p->W32 = rounded_copy(p, p->W, p->N * p->S * 4, s);
    p->Wc32 = rounded_copy(p, p->Wc, p->nnzP * 4, s);
    p->nval32 = (float2*)rounded_copy(p, (const double*)p->nval, 2 * p->nnzN, s);
    p->spec32 = (float2*)rounded_copy(p, (const double*)p->spec, 2 * p->spec_len, s);
}

void make_c64_blocks(aim_plan* p, cudaStream_t s) {
    if (p->nb_val32 || !p->nb_val) return;
    p->nb_val32 = (float2*)rounded_copy(p, (const double*)p->nb_val, 8 * p->nbc, s);
    AIM_CUDA(cudaStreamSynchronize(s));
}

void create_plan(const double* V, int64_t nv, const int32_t* T, int64_t nt, const int32_t* E, int64_t N, double k,
                 double h, int M, double r, int prec, aim_plan* p) {
    const auto t0 = std::chrono::steady_clock::now();
    AIM_CUDA(cudaGetDevice(&p->device));
    AIM_CUDA(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
    AIM_CUDA(cudaStreamCreateWithFlags(&p->side, cudaStreamNonBlocking));
    AIM_CUDA(cudaEventCreateWithFlags(&p->ev_x, cudaEventDisableTiming));
    AIM_CUDA(cudaEventCreateWithFlags(&p->ev_n, cudaEventDisableTiming));
    p->N = N; p->nt = nt; p->nv = nv; p->k = k; p->h = h; p->M = M; p->r = r;
    p->prec = prec;
    p->S = (M + 1) * (M + 1) * (M + 1);

    // ---- S0: triangle geometry + quadrature
    double bary[7][3], bw[7];
    dunavant7(bary, bw);
    std::vector<double> qp(nt * 21), qw(nt * 7), cor(nt * 9), area(nt);
    std::vector<int32_t> tv(nt * 3);
    for (int64_t t = 0; t < nt; ++t) {
        const double* P[3];
        for (int c = 0; c < 3; ++c) {
            const int32_t vi = T[3 * t + c];
            if (vi < 0 || vi >= nv) throw Error(AIM_E_MESH, "triangle vertex index out of range");
            P[c] = V + 3 * (int64_t)vi;
            tv[3 * t + c] = vi;
            for (int d = 0; d < 3; ++d) cor[9 * t + 3 * c + d] = P[c][d];
        }
        const double e1[3] = {P[1][0] - P[0][0], P[1][1] - P[0][1], P[1][2] - P[0][2]};
        const double e2[3] = {P[2][0] - P[0][0], P[2][1] - P[0][1], P[2][2] - P[0][2]};
        const double cr[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2], e1[0] * e2[1] - e1[1] * e2[0]};
        area[t] = 0.5 * sqrt(cr[0] * cr[0] + cr[1] * cr[1] + cr[2] * cr[2]);
        if (!(area[t] > 0)) throw Error(AIM_E_MESH, "degenerate triangle " + std::to_string(t));
        for (int q = 0; q < 7; ++q) {
            for (int d = 0; d < 3; ++d)
                qp[21 * t + 3 * q + d] = bary[q][0] * P[0][d] + bary[q][1] * P[1][d] + bary[q][2] * P[2][d];
            qw[7 * t + q] = bw[q] * area[t];
        }
    }
    // ---- S0: RWG geometry; Lambda = alpha (r - p), alpha = +l/(2A+) on t+, -l/(2A-) on t-
    std::vector<int32_t> rt(2 * N), base(3 * N), node0(N);
    std::vector<double> ra(2 * N), rp(6 * N), rc(3 * N);
    for (int64_t n = 0; n < N; ++n) {
        const int32_t va = E[4 * n], vb = E[4 * n + 1], tp = E[4 * n + 2], tm = E[4 * n + 3];
        if (va < 0 || va >= nv || vb < 0 || vb >= nv || va == vb)
            throw Error(AIM_E_MESH, "rwg edge vertex invalid at row " + std::to_string(n));
        if (tp < 0 || tp >= nt || tm < 0 || tm >= nt) throw Error(AIM_E_MESH, "rwg triangle index out of range");
        if (tp == tm) throw Error(AIM_E_MESH, "t+ == t- at row " + std::to_string(n));
        const double l = sqrt((V[3 * vb] - V[3 * va]) * (V[3 * vb] - V[3 * va]) +
                              (V[3 * vb + 1] - V[3 * va + 1]) * (V[3 * vb + 1] - V[3 * va + 1]) +
                              (V[3 * vb + 2] - V[3 * va + 2]) * (V[3 * vb + 2] - V[3 * va + 2]));
        const int32_t tri[2] = {tp, tm};
        double cen[3] = {0, 0, 0};
        for (int side = 0; side < 2; ++side) {
            const int32_t t = tri[side];
            int hasa = 0, hasb = 0, fv = -1;
            for (int c = 0; c < 3; ++c) {
                const int32_t v = T[3 * t + c];
                if (v == va) hasa = 1;
                else if (v == vb) hasb = 1;
                else fv = v;
            }
            if (!hasa || !hasb || fv < 0) throw Error(AIM_E_MESH, "rwg edge not in its triangle at row " + std::to_string(n));
            rt[2 * n + side] = t;
            ra[2 * n + side] = (side == 0 ? 1.0 : -1.0) * l / (2.0 * area[t]);
            for (int d = 0; d < 3; ++d) {
                rp[6 * n + 3 * side + d] = V[3 * fv + d];
                cen[d] += (V[3 * T[3 * t] + d] + V[3 * T[3 * t + 1] + d] + V[3 * T[3 * t + 2] + d]) / 3.0;
            }
        }
        for (int d = 0; d < 3; ++d) rc[3 * n + d] = 0.5 * cen[d];
    }
    // ---- S1: stencils (D3) and grid box (D4)
    long long lo[3] = {LLONG_MAX, LLONG_MAX, LLONG_MAX}, hi[3] = {LLONG_MIN, LLONG_MIN, LLONG_MIN};
    for (int64_t n = 0; n < N; ++n)
        for (int d = 0; d < 3; ++d) {
            const double s = floor(rc[3 * n + d] / h - (M - 1) / 2.0 + 1e-7);
            if (!(fabs(s) < 1e9)) throw Error(AIM_E_GRID, "stencil index exceeds addressable grid");
            const long long si = (long long)s;
            base[3 * n + d] = (int32_t)si;
            lo[d] = std::min(lo[d], si);
            hi[d] = std::max(hi[d], si);
        }
    long long ng = 1, npad = 1;
    for (int d = 0; d < 3; ++d) {
        const long long nd = hi[d] + M + 1 - lo[d];
        if (nd > (1 << 20)) throw Error(AIM_E_GRID, "grid extent exceeds addressable grid");
        p->origin[d] = (int)lo[d];
        p->dims[d] = (int)nd;
        p->pads[d] = smooth_size_at_least((int)(2 * nd - 1));
        ng *= nd;
        npad *= p->pads[d];
    }
    if (npad > 2147483647LL || ng > 2147483647LL) throw Error(AIM_E_GRID, "padded grid exceeds 2^31 points");
    if ((long long)N * p->S > 2147483647LL) throw Error(AIM_E_GRID, "projection nnz exceeds 2^31-1");
    p->Ng = ng;
    for (int64_t n = 0; n < N; ++n)
        node0[n] = (int32_t)(((long long)(base[3 * n] - lo[0]) * p->dims[1] + (base[3 * n + 1] - lo[1])) * p->dims[2] +
                             (base[3 * n + 2] - lo[2]));

    // host copies kept for the block-Jacobi preconditioner (element grouping)
    p->h_tv = tv;
    p->h_cor = cor;
    p->h_rt = rt;

    // ---- uploads
    p->tri_qp = upload(p, qp);
    p->tri_qw = upload(p, qw);
    p->tri_cor = upload(p, cor);
    p->tri_v = upload(p, tv);
    p->rwg_t = upload(p, rt);
    p->rwg_a = upload(p, ra);
    p->rwg_p = upload(p, rp);
    p->rwg_c = upload(p, rc);
    p->base = upload(p, base);
    p->node0 = upload(p, node0);
    for (int d = 0; d < 3; ++d) make_fft_axis(p->pads[d], p->ax[d]);
    // conv mode: 1 = fused planar y/z kernel (the Py x Nz plane fits shared memory),
    // 2 = thin grid with long lines: separate y passes around a z Toeplitz kernel,
    // 0 = 3-D FFT convolution.  AIM_CONV_MODE=0|1|2 forces one (tests on small grids).
    p->planar = planar_supported(p->pads[1], p->dims[2], p->ax[1].min_radix) ? 1
              : (p->dims[2] <= kPlanarMaxNz ? 2 : 0);
    if (const char* cm = getenv("AIM_CONV_MODE")) {
        if (cm[0] == '0') p->planar = 0;
        else if (cm[0] == '2' && p->dims[2] <= kPlanarMaxNz) p->planar = 2;
    }

    // ---- device setup S2-S4
    cudaStream_t s = p->stream;
    build_weights(p, s);
    build_projection_csr(p, node0, s);
    build_green_spectrum(p, s);
    build_near_list(p, s);
    build_near_values(p, s);
    if (p->prec == AIM_C64) make_c64_tables(p, s);
    AIM_CUDA(cudaStreamSynchronize(s));
    p->plan_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

void destroy_plan(aim_plan* p) {
    if (!p) return;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(p->device);
    // the plan's own work is on its streams; the caller orders (or has
    // finished) the products it queued on its streams before destroying
    for (cudaStream_t st : {p->stream, p->side, p->hi, p->hp_in, p->hp_out})
        if (st) cudaStreamSynchronize(st);
    for (auto& g : p->graphs) cudaGraphExecDestroy(g.exec);
    if (p->gx_fork) cudaEventDestroy(p->gx_fork);
    if (p->gx_join) cudaEventDestroy(p->gx_join);
    for (auto& a : p->allocs) cudaFree(a.first);
    for (int d = 0; d < 3; ++d)
        if (p->ax[d].tw) cudaFree(p->ax[d].tw);
    for (int d = 0; d < 3; ++d)
        if (p->ax[d].tw32) cudaFree(p->ax[d].tw32);
    for (auto e : p->ev_pool) cudaEventDestroy(e);
    if (p->stream) cudaStreamDestroy(p->stream);
    if (p->side) cudaStreamDestroy(p->side);
    if (p->hi) cudaStreamDestroy(p->hi);
    if (p->ev_h) cudaEventDestroy(p->ev_h);
    if (p->ev_x) cudaEventDestroy(p->ev_x);
    if (p->ev_n) cudaEventDestroy(p->ev_n);
    if (p->gm_host) cudaFreeHost(p->gm_host);
    if (p->gm_ev) cudaEventDestroy(p->gm_ev);
    if (p->hp_in) cudaStreamDestroy(p->hp_in);
    if (p->hp_out) cudaStreamDestroy(p->hp_out);
    for (int k = 0; k < 2; ++k) {
        if (p->hp_ev_in[k]) cudaEventDestroy(p->hp_ev_in[k]);
        if (p->hp_ev_mv[k]) cudaEventDestroy(p->hp_ev_mv[k]);
        if (p->hp_ev_out[k]) cudaEventDestroy(p->hp_ev_out[k]);
    }
    cudaSetDevice(cur);
    delete p;
}

}  // namespace aim

using namespace aim;

extern "C" {

int aim_plan_create(const double* vertices, int64_t nv, const int32_t* triangles, int64_t nt,
                    const int32_t* rwg_edges, int64_t n_rwg, double k, double h, int32_t M, double near_radius,
                    int32_t precision, const void* dist, aim_plan** out) {
    if (!out) return fail(AIM_E_ARG, "out is NULL");
    *out = nullptr;
    if (!vertices || !triangles || !rwg_edges) return fail(AIM_E_ARG, "NULL mesh pointer");
    if (nv < 3 || nt < 2 || n_rwg < 1) return fail(AIM_E_ARG, "empty mesh");
    if (!(k > 0) || !(h > 0) || M < 1 || M > 6 || !(near_radius >= 0))
        return fail(AIM_E_ARG, "k, h > 0, M in [1,6], near_radius >= 0 required");
    if (precision != AIM_C128 && precision != AIM_C64) return fail(AIM_E_ARG, "precision must be AIM_C128 or AIM_C64");
    if (dist) return fail(AIM_E_ARG, "dist must be NULL (single-GPU plan)");
    aim_plan* p = new aim_plan();
    const int st = guarded([&] {
        create_plan(vertices, nv, triangles, nt, rwg_edges, n_rwg, k, h, M, near_radius, precision, p);
        return AIM_OK;
    });
    if (st != AIM_OK) {
        const std::string msg = g_err;
        destroy_plan(p);
        g_err = msg;
        return st;
    }
    *out = p;
    return AIM_OK;
}

int aim_plan_destroy(aim_plan* plan) {
    return guarded([&] {
        destroy_plan(plan);
        return AIM_OK;
    });
}

int aim_plan_info(const aim_plan* p, aim_info* info) {
    if (!p || !info) return fail(AIM_E_ARG, "NULL argument");
    std::memset(info, 0, sizeof(*info));
    info->n_rwg = p->N;
    info->n_tri = p->nt;
    info->M = p->M;
    info->S = p->S;
    for (int d = 0; d < 3; ++d) {
        info->grid_origin[d] = p->origin[d];
        info->grid_dims[d] = p->dims[d];
        info->fft_dims[d] = p->pads[d];
    }
    info->n_nodes = p->Ng;
    info->nnz_proj = p->nnzP;
    info->nnz_near = p->nnzN;
    info->k = p->k;
    info->h = p->h;
    info->near_radius = p->r;
    info->device_bytes = p->device_bytes;
    info->plan_seconds = p->plan_seconds;
    info->conv_mode = p->planar;
    info->precision = p->prec;
    return AIM_OK;
}

int aim_matvec(aim_plan* p, const void* x, void* y, int32_t nrhs, void* stream) {
    if (!p || !x || !y || nrhs < 1) return fail(AIM_E_ARG, "bad argument");
    if (x == y) return fail(AIM_E_ARG, "x and y must not overlap");
    return guarded([&] {
        matvec(p, x, y, nrhs, (cudaStream_t)stream);
        return AIM_OK;
    });
}

int aim_matvec_host(aim_plan* p, const void* xh, void* yh, int32_t nrhs) {
    if (!p || !xh || !yh || nrhs < 1) return fail(AIM_E_ARG, "bad argument");
    return guarded([&] {
        const size_t bytes = (p->prec == AIM_C64 ? sizeof(float2) : sizeof(double2)) * (size_t)p->N * nrhs;
        if (p->hs_nrhs < nrhs) {
            p->release(p->hx);
            p->release(p->hy);
            p->hx = p->alloc<double2>((size_t)p->N * nrhs);
            p->hy = p->alloc<double2>((size_t)p->N * nrhs);
            p->hs_nrhs = nrhs;
        }
        cudaStream_t s = p->stream;
        AIM_CUDA(cudaMemcpyAsync(p->hx, xh, bytes, cudaMemcpyHostToDevice, s));
        matvec(p, p->hx, p->hy, nrhs, s);
        AIM_CUDA(cudaMemcpyAsync(yh, p->hy, bytes, cudaMemcpyDeviceToHost, s));
        AIM_CUDA(cudaStreamSynchronize(s));
        return AIM_OK;
    });
}

int aim_matvec_host_steps(aim_plan* p, const void* const* xs, void* const* ys, int32_t nsteps, int32_t nrhs) {
    if (!p || !xs || !ys || nrhs < 1 || nsteps < 0) return fail(AIM_E_ARG, "bad argument");
    for (int i = 0; i < nsteps; ++i)
        if (!xs[i] || !ys[i]) return fail(AIM_E_ARG, "NULL host buffer");
    return guarded([&] {
        const size_t elems = (size_t)p->N * nrhs;
        const size_t bytes = (p->prec == AIM_C64 ? sizeof(float2) : sizeof(double2)) * elems;
        // two device slots per direction; step i uses slot i % 2
        if (p->hp_nrhs < nrhs) {
            for (int k = 0; k < 2; ++k) {
                p->release(p->hp_x[k]);
                p->release(p->hp_y[k]);
                p->hp_x[k] = p->alloc<double2>(elems);
                p->hp_y[k] = p->alloc<double2>(elems);
            }
            p->hp_nrhs = nrhs;
        }
        if (!p->hp_in) {
            AIM_CUDA(cudaStreamCreateWithFlags(&p->hp_in, cudaStreamNonBlocking));
            AIM_CUDA(cudaStreamCreateWithFlags(&p->hp_out, cudaStreamNonBlocking));
            for (int k = 0; k < 2; ++k) {
                AIM_CUDA(cudaEventCreateWithFlags(&p->hp_ev_in[k], cudaEventDisableTiming));
                AIM_CUDA(cudaEventCreateWithFlags(&p->hp_ev_mv[k], cudaEventDisableTiming));
                AIM_CUDA(cudaEventCreateWithFlags(&p->hp_ev_out[k], cudaEventDisableTiming));
            }
        }
        cudaStream_t s = p->stream;
        for (int i = 0; i < nsteps; ++i) {
            const int k = i & 1;
            // copy-in of step i once step i-2's product no longer reads the slot
            if (i >= 2) AIM_CUDA(cudaStreamWaitEvent(p->hp_in, p->hp_ev_mv[k], 0));
            AIM_CUDA(cudaMemcpyAsync(p->hp_x[k], xs[i], bytes, cudaMemcpyHostToDevice, p->hp_in));
            AIM_CUDA(cudaEventRecord(p->hp_ev_in[k], p->hp_in));
            // product of step i once its x landed and step i-2's y was copied out
            AIM_CUDA(cudaStreamWaitEvent(s, p->hp_ev_in[k], 0));
            if (i >= 2) AIM_CUDA(cudaStreamWaitEvent(s, p->hp_ev_out[k], 0));
            matvec(p, p->hp_x[k], p->hp_y[k], nrhs, s);
            AIM_CUDA(cudaEventRecord(p->hp_ev_mv[k], s));
            // copy-out of step i
            AIM_CUDA(cudaStreamWaitEvent(p->hp_out, p->hp_ev_mv[k], 0));
            AIM_CUDA(cudaMemcpyAsync(ys[i], p->hp_y[k], bytes, cudaMemcpyDeviceToHost, p->hp_out));
            AIM_CUDA(cudaEventRecord(p->hp_ev_out[k], p->hp_out));
        }
        AIM_CUDA(cudaStreamSynchronize(p->hp_out));
        AIM_CUDA(cudaStreamSynchronize(s));
        return AIM_OK;
    });
}

int aim_gmres(aim_plan* p, const void* V, void* J, int32_t restart, double tol, int32_t max_iters,
              int32_t fixed_iters, int32_t* iters, double* rel_res) {
    if (!p || !V || !J || restart < 1 || !(tol >= 0)) return fail(AIM_E_ARG, "bad argument");
    if (p->prec != AIM_C128) return fail(AIM_E_ARG, "aim_gmres needs an AIM_C128 plan");
    return guarded([&] {
        int it = 0;
        double rr = 0;
        const int st = gmres(p, (const double2*)V, (double2*)J, restart, tol, max_iters, fixed_iters, &it, &rr);
        if (iters) *iters = it;
        if (rel_res) *rel_res = rr;
        return st;
    });
}

int aim_planewave_rhs(aim_plan* p, const double* khat, const double* pol, double E0_re, double E0_im, void* V,
                      void* stream) {
    if (!p || !khat || !pol || !V) return fail(AIM_E_ARG, "bad argument");
    if (p->prec != AIM_C128) return fail(AIM_E_ARG, "aim_planewave_rhs needs an AIM_C128 plan");
    return guarded([&] {
        launch_planewave(p, khat, pol, make_double2(E0_re, E0_im), (double2*)V, (cudaStream_t)stream);
        return AIM_OK;
    });
}

int aim_project(aim_plan* p, const void* x, void* Q, int32_t nrhs, void* stream) {
    if (!p || !x || !Q || nrhs < 1) return fail(AIM_E_ARG, "bad argument");
    return guarded([&] {
        launch_project(p, x, Q, nrhs, (cudaStream_t)stream);
        return AIM_OK;
    });
}

int aim_convolve(aim_plan* p, const void* Q, void* Phi, int32_t nrhs, void* stream) {
    if (!p || !Q || !Phi || nrhs < 1) return fail(AIM_E_ARG, "bad argument");
    return guarded([&] {
        ensure_workspace(p, nrhs);
        convolve(p, Q, Phi, nrhs, (cudaStream_t)stream);
        return AIM_OK;
    });
}

int aim_interpolate(aim_plan* p, const void* Phi, const void* x, void* y, int32_t nrhs, int32_t add_near,
                    void* stream) {
    if (!p || !y || nrhs < 1 || (add_near && !x) || (!Phi && !add_near)) return fail(AIM_E_ARG, "bad argument");
    return guarded([&] {
        cudaStream_t s = (cudaStream_t)stream;
        if (add_near) launch_near(p, x, y, nrhs, s);
        if (Phi) launch_interp(p, Phi, y, nrhs, add_near != 0, s);
        return AIM_OK;
    });
}

int aim_plan_export(const aim_plan* p, int32_t what, void* dst, int64_t bytes) {
    if (!p || !dst) return fail(AIM_E_ARG, "bad argument");
    return guarded([&] {
        const void* src = nullptr;
        int64_t need = 0;
        switch (what) {
            case AIM_EXPORT_BASES: src = p->base; need = 12 * p->N; break;
            case AIM_EXPORT_WEIGHTS: src = p->W; need = 32 * p->N * p->S; break;
            case AIM_EXPORT_NEAR_ROWPTR: src = p->nrow; need = 8 * (p->N + 1); break;
            case AIM_EXPORT_NEAR_COL: src = p->ncol; need = 4 * p->nnzN; break;
            case AIM_EXPORT_NEAR_VAL: src = p->nval; need = 16 * p->nnzN; break;
            case AIM_EXPORT_GREEN: src = p->spec; need = 16 * p->spec_len; break;
            case AIM_EXPORT_PROJ_ROWPTR: src = p->prow; need = 4 * (p->Ng + 1); break;
            case AIM_EXPORT_PROJ_ENT: src = p->pent; need = 4 * p->nnzP; break;
            default: throw Error(AIM_E_ARG, "unknown export id");
        }
        if (need != bytes) throw Error(AIM_E_ARG, "export size mismatch: need " + std::to_string(need));
        AIM_CUDA(cudaDeviceSynchronize());
        if (need) AIM_CUDA(cudaMemcpy(dst, src, need, cudaMemcpyDeviceToHost));
        return AIM_OK;
    });
}

int aim_profile(aim_plan* p, int32_t enable) {
    if (!p) return fail(AIM_E_ARG, "NULL plan");
    return guarded([&] {
        p->prof = enable ? 1 : 0;
        p->ev_used = 0;
        p->prof_count = 0;
        return AIM_OK;
    });
}

int aim_profile_read(aim_plan* p, double* ms, int64_t* count) {
    if (!p || !ms || !count) return fail(AIM_E_ARG, "bad argument");
    return guarded([&] {
        for (int i = 0; i < AIM_NUM_STAGES; ++i) ms[i] = 0.0;
        const size_t per = kProfEvents;
        if (p->ev_used % per) throw Error(AIM_E_ARG, "profiling events out of step");
        // (from, to) event slots of each stage, see matvec() in k_matvec.cu
        static const int from[AIM_NUM_STAGES] = {8, 1, 2, 3, 4, 5, 7};
        static const int to[AIM_NUM_STAGES] = {1, 2, 3, 4, 5, 6, 8};
        for (size_t b = 0; b < p->ev_used; b += per) {
            AIM_CUDA(cudaEventSynchronize(p->ev_pool[b + 6]));
            AIM_CUDA(cudaEventSynchronize(p->ev_pool[b + 8]));
            for (int i = 0; i < AIM_NUM_STAGES; ++i) {
                float t = 0.f;
                AIM_CUDA(cudaEventElapsedTime(&t, p->ev_pool[b + from[i]], p->ev_pool[b + to[i]]));
                ms[i] += t;
            }
        }
        *count = p->prof_count;
        p->ev_used = 0;
        p->prof_count = 0;
        return AIM_OK;
    });
}

const char* aim_last_error(void) { return g_err.c_str(); }

int64_t aim_launch_count(int32_t reset) {
    const long long v = g_launches;
    if (reset) g_launches = 0;
    return v;
}

}  // extern "C"

extern "C" {

int aim_precond_build(aim_plan* p, int32_t kind) {
    if (!p) return fail(AIM_E_ARG, "NULL plan");
    if (kind != AIM_PRECOND_NONE && kind != AIM_PRECOND_BLOCK_JACOBI) return fail(AIM_E_ARG, "unknown preconditioner");
    if (kind == AIM_PRECOND_BLOCK_JACOBI && p->prec != AIM_C128)
        return fail(AIM_E_ARG, "the preconditioner needs an AIM_C128 plan");
    return guarded([&] {
        if (kind == AIM_PRECOND_NONE) free_precond(p);
        else build_precond(p, p->stream);
        return AIM_OK;
    });
}

int aim_precond_apply(aim_plan* p, const void* x, void* y, void* stream) {
    if (!p || !x || !y || x == y) return fail(AIM_E_ARG, "bad argument");
    return guarded([&] {
        apply_precond(p, (const double2*)x, (double2*)y, (cudaStream_t)stream);
        return AIM_OK;
    });
}

int aim_precond_info(const aim_plan* p, int64_t* out) {
    if (!p || !out) return fail(AIM_E_ARG, "bad argument");
    out[0] = p->prec_on;
    out[1] = p->prec_on ? p->el_count : 0;
    out[2] = p->pc.ndistinct;
    out[3] = p->pc.maxn;
    out[4] = p->pc.bytes;
    return AIM_OK;
}

int aim_plan_compress(aim_plan* p, int32_t mode) {
    if (!p || mode < 0 || mode > 1) return fail(AIM_E_ARG, "bad argument");
    return guarded([&] {
        if (mode == 0) free_compressed(p);
        else build_compressed(p, p->stream);
        for (auto& g : p->graphs) cudaGraphExecDestroy(g.exec);   // captured the other near kernel
        p->graphs.clear();
        p->mv_warm.clear();
        return AIM_OK;
    });
}

int aim_compress_info(const aim_plan* p, int64_t* out) {
    if (!p || !out) return fail(AIM_E_ARG, "bad argument");
    out[0] = p->cmp_on;
    out[1] = p->cmp_blocks;
    out[2] = p->cmp_nnz;
    out[3] = p->nnzN;
    out[4] = p->cp_on;
    out[5] = p->cp_tpl_nnz;
    return AIM_OK;
}

int aim_plan_elements(aim_plan* p, int32_t* elem_of_rwg, int32_t* group, int32_t* n_elements) {
    if (!p || !n_elements) return fail(AIM_E_ARG, "bad argument");
    return guarded([&] {
        ensure_elements(p, p->stream);
        *n_elements = p->el_count;
        if (elem_of_rwg)
            for (int e = 0; e < p->el_count; ++e)
                for (int64_t q = p->el_rptr_h[e]; q < p->el_rptr_h[e + 1]; ++q) elem_of_rwg[p->el_rows_h[q]] = e;
        if (group)
            for (int e = 0; e < p->el_count; ++e) group[e] = p->el_group_h[e];
        return AIM_OK;
    });
}

int aim_reduced_set(aim_plan* p, int32_t n_types, const int32_t* nhat, const int32_t* nint, const void* D,
                    const void* T, const void* A, const void* B, const int32_t* elem_type, int32_t n_elements) {
    if (!p || n_types < 1 || !nhat || !nint || !D || !T || !A || !B || !elem_type || n_elements < 1)
        return fail(AIM_E_ARG, "bad argument");
    if (p->prec != AIM_C128) return fail(AIM_E_ARG, "the reduced system needs an AIM_C128 plan");
    return guarded([&] {
        reduced_set(p, n_types, nhat, nint, (const double2*)D, (const double2*)T, (const double2*)A,
                    (const double2*)B, elem_type, n_elements);
        return AIM_OK;
    });
}

int aim_reduced_matvec(aim_plan* p, const void* Y, void* out, void* stream) {
    if (!p || !Y || !out || Y == out) return fail(AIM_E_ARG, "bad argument");
    return guarded([&] {
        reduced_matvec(p, (const double2*)Y, (double2*)out, (cudaStream_t)stream);
        return AIM_OK;
    });
}

int aim_reduced_gmres(aim_plan* p, const void* V, void* E, int32_t restart, double tol, int32_t max_iters,
                      int32_t fixed_iters, int32_t* iters, double* rel_res) {
    if (!p || !V || !E || restart < 1 || !(tol >= 0)) return fail(AIM_E_ARG, "bad argument");
    if (!p->rd_on) return fail(AIM_E_ARG, "no reduced system set (aim_reduced_set)");
    return guarded([&] {
        GmresOps ops;
        ops.n = p->N;
        ops.matvec = [p](const double2* in, double2* o, cudaStream_t st) { reduced_matvec(p, in, o, st); };
        int it = 0;
        double rr = 0;
        const int st = gmres_core(p, ops, (const double2*)V, (double2*)E, restart, tol, max_iters, fixed_iters,
                                  &it, &rr);
        if (iters) *iters = it;
        if (rel_res) *rel_res = rr;
        return st;
    });
}

int aim_gmres_history(const aim_plan* p, double* out, int32_t cap, int32_t* count) {
    if (!p || !count || cap < 0 || (cap > 0 && !out)) return fail(AIM_E_ARG, "bad argument");
    const int32_t n = (int32_t)p->gm_hist.size();
    for (int32_t i = 0; i < std::min(n, cap); ++i) out[i] = p->gm_hist[i];
    *count = n;
    return AIM_OK;
}

}  // extern "C"
