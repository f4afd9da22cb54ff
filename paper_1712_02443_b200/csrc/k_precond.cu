// Block-Jacobi preconditioner for GMRES.
//
// The paper preconditions its GMRES solves ("solved iteratively using GMRES
// with an ILU-2 preconditioner", §VI-A)
// substitutes per-element dense block solves.  This build uses the latter
// (reading D18): the mesh's connected surfaces are the array
// elements (the equivalent surfaces), and
//     M = blockdiag_e ( Z_ex_sym[e, e] ),
// the exact symmetrised Galerkin EFIE entries (D8, D9) between all RWG pairs
// of element e.  Elements that are translates of one another (same local
// topology, corners equal up to 1e-9 of the element size after removing the
// translation) share one block, computed from the first such element -- the
// paper's reuse of identical elements, "only need to be calculated once for
// each distinct element".  Each distinct block is inverted
// on the device (batched Gauss-Jordan, partial pivoting); applying M^-1 is a
// GEMM over the elements that share an inverse (rows x elements tiles) or a
// GEMV per element when an inverse is used by few elements.
#include <math.h>

#include <algorithm>
#include <cstring>
#include <numeric>
#include <vector>

#include "aim_internal.cuh"

namespace aim {

void fill_exact_block(aim_plan* p, const int32_t* d_rows, int n, double2* d_out, cudaStream_t s);

struct GjBlk {
    long long off;   // element offset of the block in pc_inv (row-major n x n)
    int n;
    int poff;        // offset of the block's pivot rows / saved column
};

// ---------------------------------------------------- Gauss-Jordan inverse
// Step k, one CTA per block: pivot row p = argmax_{i >= k} |A[i][k]|^2 (ties:
// smallest i), swap rows k and p, save column k (f_i = A[i][k], i != k) and
// zero it, scale row k by 1/A[k][k] with A[k][k] := 1/A[k][k].
__global__ void __launch_bounds__(256) gj_pivot_kernel(const GjBlk* __restrict__ blk, double2* __restrict__ A0,
                                                       int k, int32_t* __restrict__ perm,
                                                       double2* __restrict__ colk, int* __restrict__ bad) {
    const GjBlk b = blk[blockIdx.x];
    if (k >= b.n) return;
    double2* A = A0 + b.off;
    const int n = b.n;
    __shared__ double sv[256];
    __shared__ int si[256];
    double best = -1.0;
    int bi = n;
    for (int i = k + threadIdx.x; i < n; i += blockDim.x) {
        const double2 v = A[(long long)i * n + k];
        const double m = v.x * v.x + v.y * v.y;
        if (m > best) { best = m; bi = i; }
    }
    sv[threadIdx.x] = best;
    si[threadIdx.x] = bi;
    __syncthreads();
    for (int w = blockDim.x / 2; w; w >>= 1) {
        if (threadIdx.x < w) {
            const double o = sv[threadIdx.x + w];
            const int oi = si[threadIdx.x + w];
            if (o > sv[threadIdx.x] || (o == sv[threadIdx.x] && oi < si[threadIdx.x])) {
                sv[threadIdx.x] = o;
                si[threadIdx.x] = oi;
            }
        }
        __syncthreads();
    }
    const int p = si[0];
    if (threadIdx.x == 0) {
        perm[b.poff + k] = p;
        if (!(sv[0] > 0.0) || !isfinite(sv[0])) *bad = 1;
    }
    if (p != k)
        for (int j = threadIdx.x; j < n; j += blockDim.x) {
            const double2 t = A[(long long)k * n + j];
            A[(long long)k * n + j] = A[(long long)p * n + j];
            A[(long long)p * n + j] = t;
        }
    __syncthreads();
    const double2 piv = A[(long long)k * n + k];
    const double d = piv.x * piv.x + piv.y * piv.y;
    const double2 ip = make_double2(piv.x / d, -piv.y / d);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        if (i == k) continue;
        colk[b.poff + i] = A[(long long)i * n + k];
        A[(long long)i * n + k] = make_double2(0, 0);
    }
    __syncthreads();
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        const double2 v = j == k ? make_double2(1, 0) : A[(long long)k * n + j];
        A[(long long)k * n + j] = make_double2(v.x * ip.x - v.y * ip.y, v.x * ip.y + v.y * ip.x);
    }
}

// Step k elimination: A[i][j] -= f_i A[k][j] for i != k (blockIdx.y = block,
// blockIdx.x = tile of 8 rows).
__global__ void __launch_bounds__(256) gj_elim_kernel(const GjBlk* __restrict__ blk, double2* __restrict__ A0, int k,
                                                      const double2* __restrict__ colk) {
    const GjBlk b = blk[blockIdx.y];
    if (k >= b.n) return;
    const int n = b.n;
    const int i0 = blockIdx.x * 8;
    if (i0 >= n) return;
    double2* A = A0 + b.off;
    const double2* rk = A + (long long)k * n;
    for (int r = 0; r < 8; ++r) {
        const int i = i0 + r;
        if (i >= n) break;
        if (i == k) continue;
        const double2 f = colk[b.poff + i];
        double2* ri = A + (long long)i * n;
        for (int j = threadIdx.x; j < n; j += blockDim.x) {
            const double2 a = rk[j];
            double2 v = ri[j];
            v.x -= f.x * a.x - f.y * a.y;
            v.y -= f.x * a.y + f.y * a.x;
            ri[j] = v;
        }
    }
}

// Undo the row interchanges as column interchanges, k = n-1 .. 0.
__global__ void __launch_bounds__(256) gj_unperm_kernel(const GjBlk* __restrict__ blk, double2* __restrict__ A0,
                                                        const int32_t* __restrict__ perm) {
    const GjBlk b = blk[blockIdx.x];
    double2* A = A0 + b.off;
    const int n = b.n;
    for (int k = n - 1; k >= 0; --k) {
        const int p = perm[b.poff + k];
        if (p != k)
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                const double2 t = A[(long long)i * n + k];
                A[(long long)i * n + k] = A[(long long)i * n + p];
                A[(long long)i * n + p] = t;
            }
        __syncthreads();
    }
}

// --------------------------------------------------------------- apply
// Shared block (GEMM): out[rows_e[i]] (+)= sum_j Blk[i][j] in[rows_e[j]] for
// the elements e of list `el` (all of size n).  CTA tile: 64 rows x 64
// elements, k-chunks of 8; thread (tr, tc) owns rows tr + 16 a, elements
// tc + 16 b (a, b < 4): 16 complex accumulators.
constexpr int kPcTile = 64, kPcK = 8;
__global__ void __launch_bounds__(256) pc_gemm_kernel(const double2* __restrict__ Blk, int n,
                                                      const int32_t* __restrict__ el, int m,
                                                      const int32_t* __restrict__ rows,
                                                      const int64_t* __restrict__ rptr,
                                                      const double2* __restrict__ in, double2* __restrict__ out,
                                                      int accumulate) {
    __shared__ double2 As[kPcK][kPcTile + 1];
    __shared__ double2 Bs[kPcK][kPcTile + 1];
    __shared__ long long rbase[kPcTile];
    const int tr = threadIdx.x & 15, tc = threadIdx.x >> 4;
    const int i0 = blockIdx.x * kPcTile, e0 = blockIdx.y * kPcTile;
    if (threadIdx.x < kPcTile) {
        const int e = e0 + threadIdx.x;
        rbase[threadIdx.x] = e < m ? rptr[el[e]] : -1;
    }
    double2 acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = make_double2(0, 0);
    __syncthreads();
    for (int j0 = 0; j0 < n; j0 += kPcK) {
        for (int t = threadIdx.x; t < kPcK * kPcTile; t += 256) {
            const int r = t / kPcK, c = t - (t / kPcK) * kPcK;
            const int i = i0 + r, j = j0 + c;
            As[c][r] = (i < n && j < n) ? __ldg(&Blk[(long long)i * n + j]) : make_double2(0, 0);
            const int cc = t / kPcTile, ee = t - (t / kPcTile) * kPcTile;
            const int jj = j0 + cc;
            const long long rb = rbase[ee];
            Bs[cc][ee] = (rb >= 0 && jj < n) ? __ldg(&in[rows[rb + jj]]) : make_double2(0, 0);
        }
        __syncthreads();
#pragma unroll
        for (int c = 0; c < kPcK; ++c) {
            double2 av[4], bv[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) av[a] = As[c][tr + 16 * a];
#pragma unroll
            for (int b = 0; b < 4; ++b) bv[b] = Bs[c][tc + 16 * b];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    acc[a][b].x = fma(av[a].x, bv[b].x, fma(-av[a].y, bv[b].y, acc[a][b].x));
                    acc[a][b].y = fma(av[a].x, bv[b].y, fma(av[a].y, bv[b].x, acc[a][b].y));
                }
        }
        __syncthreads();
    }
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        const long long rb = rbase[tc + 16 * b];
        if (rb < 0) continue;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const int i = i0 + tr + 16 * a;
            if (i >= n) continue;
            double2* o = &out[rows[rb + i]];
            if (accumulate) *o = make_double2(o->x + acc[a][b].x, o->y + acc[a][b].y);
            else *o = acc[a][b];
        }
    }
}

// Few elements per block (GEMV): one CTA per (element, 64-row tile); the
// element's input is staged in shared memory, warp per row.
__global__ void __launch_bounds__(256) pc_gemv_kernel(const double2* __restrict__ mats,
                                                      const int64_t* __restrict__ off,
                                                      const int32_t* __restrict__ map,
                                                      const int32_t* __restrict__ el, const int32_t* __restrict__ rows,
                                                      const int64_t* __restrict__ rptr,
                                                      const double2* __restrict__ in, double2* __restrict__ out,
                                                      int accumulate) {
    extern __shared__ double2 xs[];
    const int e = el[blockIdx.y];
    const long long r0 = rptr[e];
    const int n = (int)(rptr[e + 1] - r0);
    const int i0 = blockIdx.x * 64;
    if (i0 >= n) return;
    const double2* Blk = mats + off[map[e]];
    for (int j = threadIdx.x; j < n; j += blockDim.x) xs[j] = __ldg(&in[rows[r0 + j]]);
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int i = i0 + w; i < min(n, i0 + 64); i += 8) {
        const double2* ri = Blk + (long long)i * n;
        double2 s = make_double2(0, 0);
        for (int j = lane; j < n; j += 32) {
            const double2 a = __ldcs(&ri[j]), x = xs[j];
            s.x = fma(a.x, x.x, fma(-a.y, x.y, s.x));
            s.y = fma(a.x, x.y, fma(a.y, x.x, s.y));
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            s.x += __shfl_xor_sync(0xffffffffu, s.x, o);
            s.y += __shfl_xor_sync(0xffffffffu, s.y, o);
        }
        if (lane == 0) {
            double2* d = &out[rows[r0 + i]];
            if (accumulate) *d = make_double2(d->x + s.x, d->y + s.y);
            else *d = s;
        }
    }
}

// Plain row-major complex GEMM C = A B (setup only: K = T A^-1 B of the
// reduced system).  Tile 64 x 64, k-chunks of 8, 16 accumulators per thread.
__global__ void __launch_bounds__(256) zgemm_rm_kernel(const double2* __restrict__ A, const double2* __restrict__ B,
                                                       double2* __restrict__ C, int m, int n, int k) {
    __shared__ double2 As[kPcK][kPcTile + 1];
    __shared__ double2 Bs[kPcK][kPcTile + 1];
    const int tr = threadIdx.x & 15, tc = threadIdx.x >> 4;
    const int i0 = blockIdx.x * kPcTile, j0c = blockIdx.y * kPcTile;
    double2 acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = make_double2(0, 0);
    for (int q0 = 0; q0 < k; q0 += kPcK) {
        for (int t = threadIdx.x; t < kPcK * kPcTile; t += 256) {
            const int r = t / kPcK, c = t - (t / kPcK) * kPcK;
            As[c][r] = (i0 + r < m && q0 + c < k) ? A[(long long)(i0 + r) * k + q0 + c] : make_double2(0, 0);
            const int cc = t / kPcTile, jj = t - (t / kPcTile) * kPcTile;
            Bs[cc][jj] = (q0 + cc < k && j0c + jj < n) ? B[(long long)(q0 + cc) * n + j0c + jj] : make_double2(0, 0);
        }
        __syncthreads();
#pragma unroll
        for (int c = 0; c < kPcK; ++c) {
            double2 av[4], bv[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) av[a] = As[c][tr + 16 * a];
#pragma unroll
            for (int b = 0; b < 4; ++b) bv[b] = Bs[c][tc + 16 * b];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    acc[a][b].x = fma(av[a].x, bv[b].x, fma(-av[a].y, bv[b].y, acc[a][b].x));
                    acc[a][b].y = fma(av[a].x, bv[b].y, fma(av[a].y, bv[b].x, acc[a][b].y));
                }
        }
        __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int i = i0 + tr + 16 * a, j = j0c + tc + 16 * b;
            if (i < m && j < n) C[(long long)i * n + j] = acc[a][b];
        }
}

void zgemm_rm(const double2* A, const double2* B, double2* C, int m, int n, int k, cudaStream_t s) {
    const dim3 grid((unsigned)((m + kPcTile - 1) / kPcTile), (unsigned)((n + kPcTile - 1) / kPcTile));
    zgemm_rm_kernel<<<grid, 256, 0, s>>>(A, B, C, m, n, k);
    note_launch("zgemm_rm");
}

// ------------------------------------------------------------- host side
namespace {
struct Uf {
    std::vector<int32_t> par;
    explicit Uf(size_t n) : par(n) { std::iota(par.begin(), par.end(), 0); }
    int32_t find(int32_t x) {
        while (par[x] != x) x = par[x] = par[par[x]];
        return x;
    }
    void unite(int32_t a, int32_t b) {
        a = find(a);
        b = find(b);
        if (a != b) par[std::max(a, b)] = std::min(a, b);
    }
};
}  // namespace

// Elements = connected surfaces (triangles joined by an RWG), ordered by
// smallest RWG id; translate groups (D18): same local topology, corners equal
// to 1e-9 of the element size after removing the translation.
void ensure_elements(aim_plan* p, cudaStream_t s) {
    if (p->el_count) return;
    const long long N = p->N, nt = p->nt;
    const int32_t* rt = p->h_rt.data();
    const int32_t* tv = p->h_tv.data();
    const double* cor = p->h_cor.data();
    Uf uf((size_t)nt);
    for (long long n = 0; n < N; ++n) uf.unite(rt[2 * n], rt[2 * n + 1]);
    std::vector<int32_t> elem_of_root((size_t)nt, -1), elem((size_t)N);
    int ne = 0;
    for (long long n = 0; n < N; ++n) {
        const int32_t r = uf.find(rt[2 * n]);
        if (elem_of_root[r] < 0) elem_of_root[r] = ne++;
        elem[n] = elem_of_root[r];
    }
    std::vector<int64_t> rptr(ne + 1, 0);
    for (long long n = 0; n < N; ++n) rptr[elem[n] + 1]++;
    for (int e = 0; e < ne; ++e) rptr[e + 1] += rptr[e];
    std::vector<int32_t> rows((size_t)N);
    {
        std::vector<int64_t> fill(rptr.begin(), rptr.end() - 1);
        for (long long n = 0; n < N; ++n) rows[fill[elem[n]]++] = (int32_t)n;
    }
    std::vector<int32_t> tmin(ne, INT32_MAX), vmin(ne, INT32_MAX);
    for (int e = 0; e < ne; ++e)
        for (int64_t q = rptr[e]; q < rptr[e + 1]; ++q)
            for (int sd = 0; sd < 2; ++sd) {
                const int32_t t = rt[2 * rows[q] + sd];
                tmin[e] = std::min(tmin[e], t);
                for (int c = 0; c < 3; ++c) vmin[e] = std::min(vmin[e], tv[3 * t + c]);
            }
    auto same = [&](int a, int b) -> bool {   // element b a translate of element a?
        if (rptr[a + 1] - rptr[a] != rptr[b + 1] - rptr[b]) return false;
        const double* oa = cor + 9LL * tmin[a];
        const double* ob = cor + 9LL * tmin[b];
        double ext = 0;
        for (int64_t q = 0; q < rptr[a + 1] - rptr[a]; ++q)
            for (int sd = 0; sd < 2; ++sd) {
                const int32_t ta = rt[2 * rows[rptr[a] + q] + sd], tb = rt[2 * rows[rptr[b] + q] + sd];
                if (ta - tmin[a] != tb - tmin[b]) return false;
                for (int c = 0; c < 3; ++c) {
                    if (tv[3 * ta + c] - vmin[a] != tv[3 * tb + c] - vmin[b]) return false;
                    for (int d = 0; d < 3; ++d) {
                        const double da = cor[9LL * ta + 3 * c + d] - oa[d], db = cor[9LL * tb + 3 * c + d] - ob[d];
                        ext = std::max(ext, fabs(da));
                        if (fabs(da - db) > 1e-9 * std::max(1.0, ext)) return false;
                    }
                }
            }
        return true;
    };
    std::vector<int32_t> group(ne), reps;
    for (int e = 0; e < ne; ++e) {
        int found = -1;
        for (size_t r = 0; r < reps.size() && found < 0; ++r)
            if (same(reps[r], e)) found = (int)r;
        if (found < 0) {
            found = (int)reps.size();
            reps.push_back(e);
        }
        group[e] = found;
    }
    p->el_rows = p->alloc<int32_t>(N);
    p->el_rptr = p->alloc<int64_t>(ne + 1);
    h2d(p->el_rows, rows.data(), sizeof(int32_t) * N, s);
    h2d(p->el_rptr, rptr.data(), sizeof(int64_t) * (ne + 1), s);
    p->el_rows_h = std::move(rows);
    p->el_rptr_h = std::move(rptr);
    p->el_group_h = std::move(group);
    p->el_reps_h = std::move(reps);
    p->el_count = ne;
}

void invert_blocks(double2* mats, const std::vector<int64_t>& off_h, const std::vector<int>& sizes, cudaStream_t s) {
    const int nd = (int)sizes.size();
    if (!nd) return;
    std::vector<GjBlk> blk(nd);
    int maxn = 0, poff = 0;
    for (int d = 0; d < nd; ++d) {
        blk[d] = GjBlk{off_h[d], sizes[d], poff};
        poff += sizes[d];
        maxn = std::max(maxn, sizes[d]);
    }
    GjBlk* dblk = nullptr;
    int32_t* perm = nullptr;
    double2* colk = nullptr;
    int* bad = nullptr;
    AIM_CUDA(cudaMalloc(&dblk, sizeof(GjBlk) * nd));
    AIM_CUDA(cudaMalloc(&perm, sizeof(int32_t) * poff));
    AIM_CUDA(cudaMalloc(&colk, sizeof(double2) * poff));
    AIM_CUDA(cudaMalloc(&bad, sizeof(int)));
    AIM_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), s));
    AIM_CUDA(cudaMemcpyAsync(dblk, blk.data(), sizeof(GjBlk) * nd, cudaMemcpyHostToDevice, s));
    for (int k = 0; k < maxn; ++k) {
        gj_pivot_kernel<<<nd, 256, 0, s>>>(dblk, mats, k, perm, colk, bad);
        note_launch("gj_pivot");
        gj_elim_kernel<<<dim3((maxn + 7) / 8, nd), 256, 0, s>>>(dblk, mats, k, colk);
        note_launch("gj_elim");
    }
    gj_unperm_kernel<<<nd, 256, 0, s>>>(dblk, mats, perm);
    note_launch("gj_unperm");
    int hbad = 0;
    AIM_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
    AIM_CUDA(cudaStreamSynchronize(s));
    cudaFree(dblk);
    cudaFree(perm);
    cudaFree(colk);
    cudaFree(bad);
    if (hbad) throw Error(AIM_E_BREAKDOWN, "Gauss-Jordan: a singular or non-finite block");
}

void free_blocks(aim_plan* p, BlockSet& b) {
    p->release(b.mats);
    p->release(b.off);
    p->release(b.map);
    p->release(b.elist);
    b = BlockSet{};
}

void setup_block_apply(aim_plan* p, BlockSet& b, const std::vector<int32_t>& map, const std::vector<int>& sizes,
                       cudaStream_t s) {
    const int ne = p->el_count, nd = (int)sizes.size();
    b.ndistinct = nd;
    b.maxn = 0;
    for (int d = 0; d < nd; ++d) b.maxn = std::max(b.maxn, sizes[d]);
    b.map = p->alloc<int32_t>(ne);
    h2d(b.map, map.data(), sizeof(int32_t) * ne, s);
    std::vector<int64_t> off(nd + 1, 0);
    for (int d = 0; d < nd; ++d) off[d + 1] = off[d] + (int64_t)sizes[d] * sizes[d];
    std::vector<std::vector<int32_t>> users(nd);
    for (int e = 0; e < ne; ++e) users[map[e]].push_back(e);
    std::vector<int32_t> elist, gemv;
    b.jobs.clear();
    for (int d = 0; d < nd; ++d) {
        if (users[d].size() >= 8) {
            b.jobs.push_back({d, (int)elist.size(), (int)users[d].size(), sizes[d], off[d]});
            elist.insert(elist.end(), users[d].begin(), users[d].end());
        } else {
            gemv.insert(gemv.end(), users[d].begin(), users[d].end());
        }
    }
    b.gemv_off = (int)elist.size();
    b.gemv_cnt = (int)gemv.size();
    elist.insert(elist.end(), gemv.begin(), gemv.end());
    b.elist = p->alloc<int32_t>(std::max<size_t>(1, elist.size()));
    if (!elist.empty()) h2d(b.elist, elist.data(), sizeof(int32_t) * elist.size(), s);
    b.bytes = 16 * off[nd];
}

void apply_blocks(aim_plan* p, const BlockSet& b, const double2* in, double2* out, bool accumulate, cudaStream_t s) {
    for (const auto& j : b.jobs) {
        const dim3 grid((unsigned)((j.n + kPcTile - 1) / kPcTile), (unsigned)((j.m + kPcTile - 1) / kPcTile));
        pc_gemm_kernel<<<grid, 256, 0, s>>>(b.mats + j.ioff, j.n, b.elist + j.eoff, j.m, p->el_rows, p->el_rptr, in,
                                            out, accumulate ? 1 : 0);
        note_launch("blk_gemm");
    }
    if (b.gemv_cnt) {
        const size_t smem = sizeof(double2) * b.maxn;
        static unsigned long long attr_mask = 0;   // per device: the attribute is per device
        if (smem > 48 * 1024 && !(attr_mask >> (p->device & 63) & 1ULL)) {
            AIM_CUDA(cudaFuncSetAttribute(pc_gemv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
            attr_mask |= 1ULL << (p->device & 63);
        }
        const dim3 grid((unsigned)((b.maxn + 63) / 64), (unsigned)b.gemv_cnt);
        pc_gemv_kernel<<<grid, 256, smem, s>>>(b.mats, b.off, b.map, b.elist + b.gemv_off, p->el_rows, p->el_rptr,
                                               in, out, accumulate ? 1 : 0);
        note_launch("blk_gemv");
    }
}

// ------------------------------------------------------ block-Jacobi (D18)
void free_precond(aim_plan* p) {
    free_blocks(p, p->pc);
    p->prec_on = 0;
}

void build_precond(aim_plan* p, cudaStream_t s) {
    free_precond(p);
    ensure_elements(p, s);
    const int nd = (int)p->el_reps_h.size();
    std::vector<int> sizes(nd);
    std::vector<int64_t> off(nd + 1, 0);
    for (int d = 0; d < nd; ++d) {
        const int r = p->el_reps_h[d];
        sizes[d] = (int)(p->el_rptr_h[r + 1] - p->el_rptr_h[r]);
        off[d + 1] = off[d] + (int64_t)sizes[d] * sizes[d];
    }
    BlockSet& b = p->pc;
    b.mats = p->alloc<double2>(std::max<int64_t>(1, off[nd]));
    b.off = p->alloc<int64_t>(nd + 1);
    h2d(b.off, off.data(), sizeof(int64_t) * (nd + 1), s);
    // dense blocks Z_ex_sym of the representatives, inverted in place
    for (int d = 0; d < nd; ++d)
        fill_exact_block(p, p->el_rows + p->el_rptr_h[p->el_reps_h[d]], sizes[d], b.mats + off[d], s);
    try {
        invert_blocks(b.mats, off, sizes, s);
    } catch (...) {
        free_precond(p);
        throw;
    }
    setup_block_apply(p, b, p->el_group_h, sizes, s);
    p->prec_on = 1;
}

void apply_precond(aim_plan* p, const double2* in, double2* out, cudaStream_t s) {
    if (!p->prec_on) throw Error(AIM_E_ARG, "no preconditioner built (aim_precond_build)");
    apply_blocks(p, p->pc, in, out, false, s);
}

}  // namespace aim
