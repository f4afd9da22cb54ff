// Repetition-compressed near field.
//
// "In most array problems, many elements are identical.  Therefore, matrices
// T_m, A_m and B_m only need to be calculated once for each distinct element"
// (also PAPER.md:77-78).  Applied to the AIM operator: on a
// grid-commensurate lattice (elements that are translates of one another by
// integer multiples of h, so their stencils sit identically on the grid), the
// precorrected near-field block between elements e and f depends only on
// (group(e), group(f), lattice offset of f from e).  One dictionary block is
// kept per such key (the entries of its first occurrence in element order);
// every element lists its neighbour elements with the key of each pair.  The
// product walks, for row m (element e, local row l), the neighbour slots of e
// and the dictionary row l of each slot's block, gathering x of the
// neighbour's RWGs.  C4: 478 M stored entries -> the dictionary of a few
// blocks (L2-resident); the structure of every occurrence is verified equal
// to its block's at build time.
#include <algorithm>
#include <cstdlib>
#include <map>
#include <tuple>
#include <vector>

#include "aim_internal.cuh"
#include "cplx.cuh"

namespace aim {

__global__ void cz_gather_kernel(const double2* __restrict__ src, const int64_t* __restrict__ idx, long long n,
                                 double2* __restrict__ dst) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[idx[i]];
}

// y[m] (+)= sum_slots sum_{entries of block row l} val * x[rwg(f, l')], warp per
// row (rows walked element-major so a CTA's warps share neighbour blocks in L1)
template <class C>
__global__ void __launch_bounds__(256) near_cmp_kernel(const int32_t* __restrict__ el_rows,
                                                       const int64_t* __restrict__ el_rptr,
                                                       const int32_t* __restrict__ el_of,
                                                       const int32_t* __restrict__ loc,
                                                       const int64_t* __restrict__ slot_ptr,
                                                       const int32_t* __restrict__ slot_f,
                                                       const int32_t* __restrict__ slot_b,
                                                       const int64_t* __restrict__ brow,
                                                       const int64_t* __restrict__ rowptr,
                                                       const int32_t* __restrict__ col, const C* __restrict__ val,
                                                       int contig, const C* __restrict__ x, long long N, int R,
                                                       C* __restrict__ y) {
    const long long q = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / 32;
    if (q >= N) return;
    const int lane = threadIdx.x & 31;
    const int m = el_rows[q];
    const int e = el_of[m], l = loc[m];
    for (int r = 0; r < R; ++r) {
        C acc = mkc<C>(0, 0);
        for (long long sl = slot_ptr[e]; sl < slot_ptr[e + 1]; ++sl) {
            const int f = slot_f[sl];
            const int64_t* rp = rowptr + brow[slot_b[sl]];
            const long long e0 = rp[l], e1 = rp[l + 1];
            const long long fb = el_rptr[f];
            for (long long b = e0 + lane; b < e1; b += 64) {
                C z[2], xv[2];
                int n[2];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const long long t = b + 32 * u;
                    const bool v = t < e1;
                    z[u] = v ? __ldg(&val[t]) : mkc<C>(0, 0);
                    const int lc = v ? __ldg(&col[t]) : 0;
                    n[u] = v ? (contig ? (int)(el_rows[fb] + lc) : el_rows[fb + lc]) : -1;
                }
#pragma unroll
                for (int u = 0; u < 2; ++u) xv[u] = n[u] >= 0 ? __ldg(&x[(long long)n[u] * R + r]) : mkc<C>(0, 0);
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    acc.x = fma(z[u].x, xv[u].x, acc.x); acc.x = fma(-z[u].y, xv[u].y, acc.x);
                    acc.y = fma(z[u].x, xv[u].y, acc.y); acc.y = fma(z[u].y, xv[u].x, acc.y);
                }
            }
        }
#pragma unroll
        for (int off = 16; off; off >>= 1) {
            const C t = shfl_xor2(acc, off);
            acc.x += t.x; acc.y += t.y;
        }
        if (lane == 0) y[(long long)m * R + r] = acc;
    }
}

// One right-hand side: warp per row; lanes < (number of slots) first fetch
// their slot's block row range and the neighbour's first RWG id, then the
// warp walks the slots with that metadata in registers (shuffles, no
// dependent loads), lane t taking entries t and t + 32 of each slot's row;
// four slots are unrolled so their value / column / x loads overlap.
constexpr int kCzMaxSlots = 32;
__global__ void __launch_bounds__(256) near_cmp1_kernel(const int32_t* __restrict__ el_rows,
                                                        const int64_t* __restrict__ el_rptr,
                                                        const int32_t* __restrict__ el_of,
                                                        const int32_t* __restrict__ loc,
                                                        const int64_t* __restrict__ slot_ptr,
                                                        const int32_t* __restrict__ slot_f,
                                                        const int32_t* __restrict__ slot_b,
                                                        const int64_t* __restrict__ brow,
                                                        const int64_t* __restrict__ rowptr,
                                                        const int32_t* __restrict__ col,
                                                        const double2* __restrict__ val,
                                                        const double2* __restrict__ x, long long N,
                                                        double2* __restrict__ y) {
    const long long q = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / 32;
    if (q >= N) return;
    const int lane = threadIdx.x & 31;
    const int m = el_rows[q];
    const int e = el_of[m], l = loc[m];
    const long long s0 = slot_ptr[e];
    const int ns = (int)(slot_ptr[e + 1] - s0);
    long long st = 0;
    int cnt = 0, fb = 0;
    if (lane < ns) {
        const int64_t* rp = rowptr + brow[slot_b[s0 + lane]];
        st = rp[l];
        cnt = (int)(rp[l + 1] - st);
        fb = el_rows[el_rptr[slot_f[s0 + lane]]];
    }
    double2 acc = make_double2(0, 0);
    for (int sb = 0; sb < ns; sb += 4) {
        double2 z[4][2];
        int n[4][2];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int sl = sb + k;
            const long long st_k = __shfl_sync(0xffffffffu, st, sl & 31);
            const int cnt_k = sl < ns ? __shfl_sync(0xffffffffu, cnt, sl & 31) : 0;
            const int fb_k = __shfl_sync(0xffffffffu, fb, sl & 31);
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int t = lane + 32 * u;
                const bool v = t < cnt_k;
                z[k][u] = v ? __ldg(&val[st_k + t]) : make_double2(0, 0);
                n[k][u] = v ? fb_k + __ldg(&col[st_k + t]) : -1;
            }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const double2 xv = n[k][u] >= 0 ? __ldg(&x[n[k][u]]) : make_double2(0, 0);
                acc.x = fma(z[k][u].x, xv.x, acc.x); acc.x = fma(-z[k][u].y, xv.y, acc.x);
                acc.y = fma(z[k][u].x, xv.y, acc.y); acc.y = fma(z[k][u].y, xv.x, acc.y);
            }
        // rows with more than 64 entries in one slot (not in the BASELINE arrays)
#pragma unroll 1
        for (int k = 0; k < 4; ++k) {
            const int sl = sb + k;
            const long long st_k = __shfl_sync(0xffffffffu, st, sl & 31);
            const int cnt_k = sl < ns ? __shfl_sync(0xffffffffu, cnt, sl & 31) : 0;
            const int fb_k = __shfl_sync(0xffffffffu, fb, sl & 31);
            for (int t = 64 + lane; t < cnt_k; t += 32) {
                const double2 zz = __ldg(&val[st_k + t]);
                const double2 xv = __ldg(&x[fb_k + __ldg(&col[st_k + t])]);
                acc.x = fma(zz.x, xv.x, acc.x); acc.x = fma(-zz.y, xv.y, acc.x);
                acc.y = fma(zz.x, xv.y, acc.y); acc.y = fma(zz.y, xv.x, acc.y);
            }
        }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, off);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, off);
    }
    if (lane == 0) y[m] = acc;
}

// One element group (every element a lattice translate of the first; C2, C4,
// C5) and one right-hand side: the near product as a sparse x dense product
// per dictionary block b,  Yt[l][e_k] += sum_{l'} B[l][l'] Xt[l'][f_k]  over
// the element pairs (e_k, f_k) that use b, with x and y transposed to
// [local row][element] so each nonzero of B multiplies a contiguous run of
// elements (coalesced) instead of one scattered x value per stored entry.
// Thread (row slot, pair): 64 consecutive pairs per CTA column tile, the 4
// row slots of a CTA walk 16 rows.  (64 rows x 8 pairs per CTA, for L1 reuse
// of the Xt lines across rows, measured slower on C4: 1.06 vs 0.90 ms.)
constexpr int kSpRows = 16;
constexpr int kSpPairs = 64;
__global__ void cz_transpose_kernel(const double2* __restrict__ x, int n, int ne, int first_stride,
                                    const int32_t* __restrict__ el_first, double2* __restrict__ xt, int to_t) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long long)n * ne) return;
    const int l = (int)(t / ne), e = (int)(t - (t / ne) * ne);
    const long long g = (long long)el_first[e] + l;
    if (to_t) xt[t] = x[g];
    else ((double2*)x)[g] = xt[t];
}

__global__ void __launch_bounds__(256) near_spmm_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                                        const double2* __restrict__ val,
                                                        const int32_t* __restrict__ pe,
                                                        const int32_t* __restrict__ pf, int m, int n, int ne,
                                                        const double2* __restrict__ xt, double2* __restrict__ yt) {
    const int k = blockIdx.y * kSpPairs + (threadIdx.x % kSpPairs);
    const int e = k < m ? pe[k] : -1, f = k < m ? pf[k] : 0;
    for (int r = threadIdx.x / kSpPairs; r < kSpRows; r += 256 / kSpPairs) {
        const int l = blockIdx.x * kSpRows + r;
        if (l >= n) break;
        const long long t0 = rp[l], t1 = rp[l + 1];
        double2 acc = make_double2(0, 0);
        long long t = t0;
        for (; t + 4 <= t1; t += 4) {
            double2 v[4], xv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                v[u] = __ldg(&val[t + u]);
                xv[u] = __ldg(&xt[(long long)__ldg(&col[t + u]) * ne + f]);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                acc.x = fma(v[u].x, xv[u].x, acc.x); acc.x = fma(-v[u].y, xv[u].y, acc.x);
                acc.y = fma(v[u].x, xv[u].y, acc.y); acc.y = fma(v[u].y, xv[u].x, acc.y);
            }
        }
        for (; t < t1; ++t) {
            const double2 v = __ldg(&val[t]), xv = __ldg(&xt[(long long)__ldg(&col[t]) * ne + f]);
            acc.x = fma(v.x, xv.x, acc.x); acc.x = fma(-v.y, xv.y, acc.x);
            acc.y = fma(v.x, xv.y, acc.y); acc.y = fma(v.y, xv.x, acc.y);
        }
        if (e >= 0) {
            double2* o = &yt[(long long)l * ne + e];
            *o = make_double2(o->x + acc.x, o->y + acc.y);
        }
    }
}

// ------------------------------------------------ projection / interpolation
// The weights of RWG m depend only on the positions of its quadrature points
// relative to its stencil base (D2, D3), so a translate of an element by an
// integer multiple of h has the weights of its group representative, with the
// stencils shifted by the translation.  Group d's template T_d lists, per node
// p of the representative's stencil box, the pairs (local row l, stencil
// node u) with base(l) - b + off(u) = p and their four weights.  Projection:
//   1. Xt_d[l][k] = x[rwg(E_d[k], l)]         (x of the group's elements, transposed)
//   2. Qt_d[p][k][c] = sum_{t in T_d[p]} w^c_t Xt_d[l_t][k]
//      -- sparse (template) x dense (elements) product: a warp takes one box
//      node and 32 elements, the template entries are warp-uniform loads and
//      the Xt rows coalesced, so the template is read once per 64 elements;
//   3. Q^c[g] = sum_{e : g in box(e)} Qt[g - b_e][e][c], elements ascending
//      (fixed order: deterministic), one thread per grid node, the elements
//      whose box meets the CTA's 256 nodes listed per chunk.
__global__ void cp_xt_kernel(const double2* __restrict__ x, const int32_t* __restrict__ gel, int ne_d, int n_d,
                             const int32_t* __restrict__ xfirst, const int32_t* __restrict__ el_rows, int contig,
                             double2* __restrict__ xt) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long long)n_d * ne_d) return;
    const int l = (int)(t / ne_d), k = (int)(t - (long long)l * ne_d);
    const int e = gel[k];
    xt[t] = __ldg(&x[contig ? xfirst[e] + l : __ldg(&el_rows[xfirst[e] + l])]);
}

constexpr int kCpK = 64;    // elements per CTA column
constexpr int kCpP = 4;     // box nodes per CTA
__global__ void __launch_bounds__(256) cp_spmm_kernel(const int32_t* __restrict__ tptr, const int32_t* __restrict__ tl,
                                                      const double* __restrict__ tw, int nodes, int ne_d,
                                                      const double2* __restrict__ xt, double2* __restrict__ qt) {
    const int p = blockIdx.y * kCpP + (threadIdx.x / kCpK);
    const int k = blockIdx.x * kCpK + (threadIdx.x % kCpK);
    if (p >= nodes) return;
    const bool live = k < ne_d;
    const int t0 = tptr[p], t1 = tptr[p + 1];
    double2 a[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) a[c] = make_double2(0, 0);
#pragma unroll 4
    for (int t = t0; t < t1; ++t) {
        const int l = __ldg(&tl[t]);
        double w0, w1, w2, w3;
        asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];\n"
            : "=d"(w0), "=d"(w1), "=d"(w2), "=d"(w3)
            : "l"(tw + 4 * (long long)t));
        const double2 xv = live ? __ldg(&xt[(long long)l * ne_d + k]) : make_double2(0, 0);
        a[0].x = fma(w0, xv.x, a[0].x); a[0].y = fma(w0, xv.y, a[0].y);
        a[1].x = fma(w1, xv.x, a[1].x); a[1].y = fma(w1, xv.y, a[1].y);
        a[2].x = fma(w2, xv.x, a[2].x); a[2].y = fma(w2, xv.y, a[2].y);
        a[3].x = fma(w3, xv.x, a[3].x); a[3].y = fma(w3, xv.y, a[3].y);
    }
    if (live) {
        double2* o = qt + ((long long)p * ne_d + k) * 4;
#pragma unroll
        for (int c = 0; c < 4; ++c) o[c] = a[c];
    }
}

__global__ void __launch_bounds__(256) cp_gather_sum_kernel(
    const int64_t* __restrict__ cptr, const int32_t* __restrict__ cel, const int4* __restrict__ ebox,
    const int4* __restrict__ gdim, const int64_t* __restrict__ qbase, const int32_t* __restrict__ qstride,
    const double2* __restrict__ qt, int Ny, int Nz, long long Ng, double2* __restrict__ Q) {
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = g < Ng;
    const int iz = (int)(g % Nz);
    const long long gy = g / Nz;
    const int iy = (int)(gy % Ny), ix = (int)(gy / Ny);
    double2 a[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) a[c] = make_double2(0, 0);
    const long long c1 = cptr[blockIdx.x + 1];
    for (long long c = cptr[blockIdx.x]; c < c1; ++c) {
        const int e = cel[c];
        const int4 eb = ebox[e];
        const int4 gd = gdim[eb.w];
        const int px = ix - eb.x, py = iy - eb.y, pz = iz - eb.z;
        if (!live || px < 0 || py < 0 || pz < 0 || px >= gd.x || py >= gd.y || pz >= gd.z) continue;
        const long long pl = (px * gd.y + py) * gd.z + pz;
        const double2* q = qt + qbase[e] + pl * qstride[e];
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
            const double2 v = __ldcs(&q[cc]);
            a[cc].x += v.x;
            a[cc].y += v.y;
        }
    }
    if (live)
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) __stcs(&Q[(long long)cc * Ng + g], a[cc]);
}

// rows of a row-major table (width in double2) gathered into a compact copy
__global__ void cz_gather_rows_kernel(const double2* __restrict__ src, const int32_t* __restrict__ rows, int nrows,
                                      int width, double2* __restrict__ dst) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)nrows * width) return;
    const int r = (int)(i / width), k = (int)(i - (long long)r * width);
    dst[i] = src[(long long)rows[r] * width + k];
}

void launch_project_cmp(const aim_plan* p, const void* x, void* Q, cudaStream_t s) {
    for (const auto& G : p->cp_groups) {
        const long long tot = (long long)G.n * G.ne;
        cp_xt_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>((const double2*)x, p->cp_gel + G.eoff, G.ne, G.n,
                                                                   p->cp_xfirst, p->el_rows, p->cz_contig,
                                                                   p->cp_xt + G.xoff);
        note_launch("cp_xt");
        const dim3 g2((unsigned)((G.ne + kCpK - 1) / kCpK), (unsigned)((G.nodes + kCpP - 1) / kCpP));
        cp_spmm_kernel<<<g2, 256, 0, s>>>(p->cp_tptr + G.toff, p->cp_tl, p->cp_tw, G.nodes, G.ne, p->cp_xt + G.xoff,
                                          p->cp_qt + G.qoff);
        note_launch("cp_spmm");
    }
    cp_gather_sum_kernel<<<(unsigned)p->cp_chunks, 256, 0, s>>>(p->cp_cptr, p->cp_cel, p->cp_ebox, p->cp_gdim,
                                                                p->cp_qbase, p->cp_qstride, p->cp_qt, p->dims[1],
                                                                p->dims[2], p->Ng, (double2*)Q);
    note_launch("cp_gather_sum");
}

static void free_compressed_pi(aim_plan* p) {
    for (void* q : {(void*)p->cp_cptr, (void*)p->cp_cel, (void*)p->cp_ebox, (void*)p->cp_gdim, (void*)p->cp_tptr,
                    (void*)p->cp_tl, (void*)p->cp_tw, (void*)p->cp_xfirst, (void*)p->cp_wrow, (void*)p->cp_gel,
                    (void*)p->cp_qbase, (void*)p->cp_qstride, (void*)p->cp_xt, (void*)p->cp_qt})
        p->release(q);
    p->cp_cptr = p->cp_qbase = nullptr;
    p->cp_cel = p->cp_tptr = p->cp_tl = p->cp_xfirst = p->cp_wrow = p->cp_gel = p->cp_qstride = nullptr;
    p->cp_xt = p->cp_qt = nullptr;
    p->cp_groups.clear();
    p->cp_ebox = p->cp_gdim = nullptr;
    p->cp_tw = nullptr;
    p->cp_on = 0;
    p->cp_tpl_nnz = p->cp_chunks = 0;
}

// Templates, chunk lists and the interpolation's weight-row map for the
// groups of build_compressed (grp: group of every element, rep: its
// representative).  Skipped (cp_on = 0) unless the templates are at most
// half the projection CSR (AIM_CMP_PI=0 / 1 in the environment: never / always).
static void build_compressed_pi(aim_plan* p, const std::vector<int32_t>& grp, const std::vector<int32_t>& rep,
                                const std::vector<int32_t>& base, cudaStream_t s) {
    free_compressed_pi(p);
    const char* env = getenv("AIM_CMP_PI");   // 0: never, 1: whenever compressible (tests)
    if (env && env[0] == '0') return;
    const bool force = env && env[0] == '1';
    const int ne = p->el_count, ng = (int)rep.size();
    const auto& rows = p->el_rows_h;
    const auto& rptr = p->el_rptr_h;
    const int M1 = p->M + 1, S = p->S;
    int64_t tpl = 0;
    for (int d = 0; d < ng; ++d) tpl += (rptr[rep[d] + 1] - rptr[rep[d]]) * (int64_t)S;
    if ((!force && tpl * 2 > p->nnzP) || tpl >= (1LL << 31)) return;
    const int* o = p->origin;
    // element boxes: corner = smallest stencil base (grid-relative), group dims
    std::vector<int4> ebox(ne), gdim(ng);
    for (int e = 0; e < ne; ++e) {
        int lo[3] = {INT32_MAX, INT32_MAX, INT32_MAX};
        for (int64_t q = rptr[e]; q < rptr[e + 1]; ++q)
            for (int c = 0; c < 3; ++c) lo[c] = std::min(lo[c], base[3 * rows[q] + c] - o[c]);
        ebox[e] = make_int4(lo[0], lo[1], lo[2], grp[e]);
    }
    std::vector<int32_t> tptr, tl, wrow(p->N), reprows;
    std::vector<int64_t> tsrc;   // template entry -> (row of reprows) * S + u
    int64_t nrep = 0;
    for (int d = 0; d < ng; ++d) {
        const int r = rep[d];
        const int nr = (int)(rptr[r + 1] - rptr[r]);
        int hi[3] = {0, 0, 0};
        for (int l = 0; l < nr; ++l)
            for (int c = 0; c < 3; ++c) {
                const int b = base[3 * rows[rptr[r] + l] + c] - o[c] - (&ebox[r].x)[c];
                hi[c] = std::max(hi[c], b + M1);
            }
        const int B = hi[0] * hi[1] * hi[2];
        gdim[d] = make_int4(hi[0], hi[1], hi[2], (int)tptr.size());
        // counting sort of the representative's (l, u) pairs by box node
        std::vector<int32_t> cnt(B + 1, 0), node((size_t)nr * S);
        for (int l = 0; l < nr; ++l) {
            const int m = rows[rptr[r] + l];
            const int bx = base[3 * m] - o[0] - ebox[r].x, by = base[3 * m + 1] - o[1] - ebox[r].y,
                      bz = base[3 * m + 2] - o[2] - ebox[r].z;
            for (int u = 0; u < S; ++u) {
                const int ui = u / (M1 * M1), uj = (u / M1) % M1, uk = u % M1;
                const int pl = ((bx + ui) * hi[1] + (by + uj)) * hi[2] + bz + uk;
                node[(size_t)l * S + u] = pl;
                cnt[pl + 1]++;
            }
        }
        for (int q = 0; q < B; ++q) cnt[q + 1] += cnt[q];
        const int32_t t0 = (int32_t)tl.size();
        for (int q = 0; q <= B; ++q) tptr.push_back(t0 + cnt[q]);
        tl.resize(t0 + (size_t)nr * S);
        tsrc.resize(t0 + (size_t)nr * S);
        for (int l = 0; l < nr; ++l)
            for (int u = 0; u < S; ++u) {
                const int t = t0 + cnt[node[(size_t)l * S + u]]++;
                tl[t] = l;
                tsrc[t] = (nrep + l) * S + u;
            }
        for (int l = 0; l < nr; ++l) reprows.push_back(rows[rptr[r] + l]);
        nrep += nr;
    }
    // every element's stencils are its representative's shifted by its box corner
    for (int e = 0; e < ne; ++e) {
        const int r = rep[grp[e]];
        for (int64_t l = 0; l < rptr[e + 1] - rptr[e]; ++l) {
            const int m = rows[rptr[e] + l], mr = rows[rptr[r] + l];
            for (int c = 0; c < 3; ++c)
                if (base[3 * m + c] - (&ebox[e].x)[c] != base[3 * mr + c] - (&ebox[r].x)[c])
                    throw Error(AIM_E_ARG, "projection not repetition-compressible (element " + std::to_string(e) + ")");
            wrow[m] = mr;
        }
    }
    // chunks of 256/G consecutive grid nodes and the elements whose box meets them
    const int npc = 256;
    const int64_t nch = (p->Ng + npc - 1) / npc;
    std::vector<std::vector<int32_t>> lists(nch);
    const int Ny = p->dims[1], Nz = p->dims[2];
    for (int e = 0; e < ne; ++e) {
        const int4 b = ebox[e], d = gdim[grp[e]];
        for (int ix = b.x; ix < b.x + d.x; ++ix)
            for (int iy = b.y; iy < b.y + d.y; ++iy) {
                const int64_t g0 = ((int64_t)ix * Ny + iy) * Nz + b.z, g1 = g0 + d.z - 1;
                for (int64_t c = g0 / npc; c <= g1 / npc; ++c)
                    if (lists[c].empty() || lists[c].back() != e) lists[c].push_back(e);
            }
    }
    std::vector<int64_t> cptr(nch + 1, 0);
    std::vector<int32_t> cel;
    for (int64_t c = 0; c < nch; ++c) {
        cel.insert(cel.end(), lists[c].begin(), lists[c].end());
        cptr[c + 1] = (int64_t)cel.size();
    }
    std::vector<int32_t> xfirst(ne);
    for (int e = 0; e < ne; ++e) xfirst[e] = p->cz_contig ? rows[rptr[e]] : (int32_t)rptr[e];
    auto up32 = [&](const std::vector<int32_t>& v) {
        int32_t* dp = p->alloc<int32_t>(std::max<size_t>(1, v.size()));
        if (!v.empty()) h2d(dp, v.data(), sizeof(int32_t) * v.size(), s);
        return dp;
    };
    p->cp_cptr = p->alloc<int64_t>(nch + 1);
    h2d(p->cp_cptr, cptr.data(), sizeof(int64_t) * (nch + 1), s);
    p->cp_cel = up32(cel);
    p->cp_ebox = p->alloc<int4>(ne);
    h2d(p->cp_ebox, ebox.data(), sizeof(int4) * ne, s);
    p->cp_gdim = p->alloc<int4>(ng);
    h2d(p->cp_gdim, gdim.data(), sizeof(int4) * ng, s);
    p->cp_tptr = up32(tptr);
    p->cp_tl = up32(tl);
    p->cp_xfirst = up32(xfirst);
    p->cp_wrow = up32(wrow);
    // template weights: the representatives' weight rows gathered, then placed
    // in template order on the host
    {
        int32_t* d_rows = up32(reprows);
        double2* d_w = p->alloc<double2>((size_t)nrep * S * 2);
        const long long tot = nrep * (long long)S * 2;
        cz_gather_rows_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>((const double2*)p->W, d_rows, (int)nrep,
                                                                           2 * S, d_w);
        note_launch("cz_gather_rows");
        std::vector<double> wr((size_t)nrep * S * 4), tw(tl.size() * 4);
        AIM_CUDA(cudaMemcpyAsync(wr.data(), d_w, sizeof(double) * wr.size(), cudaMemcpyDeviceToHost, s));
        AIM_CUDA(cudaStreamSynchronize(s));
        p->release(d_rows);
        p->release(d_w);
        for (size_t t = 0; t < tl.size(); ++t)
            for (int c = 0; c < 4; ++c) tw[4 * t + c] = wr[4 * tsrc[t] + c];
        p->cp_tw = p->alloc<double>(std::max<size_t>(4, tw.size()));
        if (!tw.empty()) h2d(p->cp_tw, tw.data(), sizeof(double) * tw.size(), s);
    }
    // per group: its elements (ascending), the offsets of its Xt and Qt blocks;
    // per element: where its Qt column starts and the stride between box nodes
    {
        std::vector<std::vector<int32_t>> E(ng);
        for (int e = 0; e < ne; ++e) E[grp[e]].push_back(e);
        std::vector<int32_t> gel, qstride(ne);
        std::vector<int64_t> qbase(ne);
        int64_t xoff = 0, qoff = 0;
        p->cp_groups.clear();
        for (int d = 0; d < ng; ++d) {
            aim_plan::CpGroup G;
            G.ne = (int)E[d].size();
            G.n = (int)(rptr[rep[d] + 1] - rptr[rep[d]]);
            G.nodes = gdim[d].x * gdim[d].y * gdim[d].z;
            G.toff = gdim[d].w;
            G.eoff = (int)gel.size();
            G.xoff = xoff;
            G.qoff = qoff;
            for (int k = 0; k < G.ne; ++k) {
                qbase[E[d][k]] = qoff + 4LL * k;
                qstride[E[d][k]] = 4 * G.ne;
            }
            gel.insert(gel.end(), E[d].begin(), E[d].end());
            xoff += (int64_t)G.n * G.ne;
            qoff += 4LL * G.nodes * G.ne;
            p->cp_groups.push_back(G);
        }
        p->cp_gel = up32(gel);
        p->cp_qstride = up32(qstride);
        p->cp_qbase = p->alloc<int64_t>(ne);
        h2d(p->cp_qbase, qbase.data(), sizeof(int64_t) * ne, s);
        p->cp_xt = p->alloc<double2>(std::max<int64_t>(1, xoff));
        p->cp_qt = p->alloc<double2>(std::max<int64_t>(1, qoff));
    }
    p->cp_chunks = nch;
    p->cp_tpl_nnz = (int64_t)tl.size();
    p->cp_on = 1;
}

void free_compressed(aim_plan* p) {
    for (void* q : {(void*)p->cz_el_of, (void*)p->cz_loc, (void*)p->cz_slot_ptr, (void*)p->cz_slot_f,
                    (void*)p->cz_slot_b, (void*)p->cz_brow, (void*)p->cz_rowptr, (void*)p->cz_col,
                    (void*)p->cz_val})
        p->release(q);
    p->cz_el_of = p->cz_loc = p->cz_slot_f = p->cz_slot_b = p->cz_col = nullptr;
    p->cz_slot_ptr = p->cz_brow = p->cz_rowptr = nullptr;
    p->cz_val = nullptr;
    for (void* q : {(void*)p->cz_pe, (void*)p->cz_pf, (void*)p->cz_first, (void*)p->cz_xt, (void*)p->cz_yt})
        p->release(q);
    p->cz_pe = p->cz_pf = p->cz_first = nullptr;
    p->cz_xt = p->cz_yt = nullptr;
    p->cz_pairs.clear();
    free_compressed_pi(p);
    p->cmp_on = 0;
    p->cmp_nnz = p->cmp_blocks = 0;
}

void build_compressed(aim_plan* p, cudaStream_t s) {
    if (p->prec != AIM_C128) throw Error(AIM_E_ARG, "compression needs an AIM_C128 plan");
    free_compressed(p);
    ensure_elements(p, s);
    const long long N = p->N;
    const int ne = p->el_count;
    const auto& rows = p->el_rows_h;
    const auto& rptr = p->el_rptr_h;
    std::vector<int32_t> el_of(N), loc(N), base(3 * N);
    for (int e = 0; e < ne; ++e)
        for (int64_t q = rptr[e]; q < rptr[e + 1]; ++q) {
            el_of[rows[q]] = e;
            loc[rows[q]] = (int32_t)(q - rptr[e]);
        }
    AIM_CUDA(cudaMemcpy(base.data(), p->base, sizeof(int32_t) * 3 * N, cudaMemcpyDeviceToHost));
    // groups: translate groups whose members sit on the grid like their
    // representative (stencil bases shifted by one integer vector); a member
    // that does not is its own group
    std::vector<int32_t> grp(ne), shift(3 * ne, 0);
    int ng = (int)p->el_reps_h.size();
    for (int e = 0; e < ne; ++e) {
        const int d = p->el_group_h[e], r = p->el_reps_h[d];
        grp[e] = d;
        bool ok = true;
        for (int c = 0; c < 3; ++c) shift[3 * e + c] = base[3 * rows[rptr[e]] + c] - base[3 * rows[rptr[r]] + c];
        for (int64_t l = 0; ok && l < rptr[e + 1] - rptr[e]; ++l)
            for (int c = 0; c < 3; ++c)
                if (base[3 * rows[rptr[e] + l] + c] - base[3 * rows[rptr[r] + l] + c] != shift[3 * e + c]) ok = false;
        if (!ok) {
            grp[e] = ng++;
            shift[3 * e] = shift[3 * e + 1] = shift[3 * e + 2] = 0;
        }
    }
    // general near CSR on the host (structure only)
    std::vector<int64_t> nrow(N + 1);
    std::vector<int32_t> ncol(p->nnzN);
    AIM_CUDA(cudaMemcpy(nrow.data(), p->nrow, sizeof(int64_t) * (N + 1), cudaMemcpyDeviceToHost));
    AIM_CUDA(cudaMemcpy(ncol.data(), p->ncol, sizeof(int32_t) * p->nnzN, cudaMemcpyDeviceToHost));
    struct Block {
        int ge, nrows;
        std::vector<int64_t> rowptr;   // local
        std::vector<int32_t> col;
        std::vector<int64_t> src;      // index into the general CSR
    };
    std::map<std::tuple<int, int, int, int, int>, int> key_of;
    std::vector<Block> blocks;
    std::vector<int64_t> slot_ptr(ne + 1, 0);
    std::vector<int32_t> slot_f, slot_b;
    for (int e = 0; e < ne; ++e) {
        const int ne_rows = (int)(rptr[e + 1] - rptr[e]);
        std::vector<int> fs, bs;          // this element's slots
        std::vector<char> filling;        // block first seen here (filled from e's rows)
        std::vector<int64_t> cursor;      // verification cursor per slot (entries of the block row)
        for (int l = 0; l < ne_rows; ++l) {
            const int m = rows[rptr[e] + l];
            // entries of row m grouped by neighbour element, in column order
            for (int64_t t = nrow[m]; t < nrow[m + 1]; ++t) {
                const int n = ncol[t], f = el_of[n];
                size_t k = 0;
                while (k < fs.size() && fs[k] != f) ++k;
                if (k == fs.size()) {
                    const auto key = std::make_tuple(grp[e], grp[f], shift[3 * f] - shift[3 * e],
                                                     shift[3 * f + 1] - shift[3 * e + 1],
                                                     shift[3 * f + 2] - shift[3 * e + 2]);
                    auto it = key_of.find(key);
                    int b;
                    if (it == key_of.end()) {
                        b = (int)blocks.size();
                        key_of[key] = b;
                        Block B;
                        B.ge = grp[e];
                        B.nrows = ne_rows;
                        B.rowptr.assign(ne_rows + 1, -1);
                        B.rowptr[0] = 0;
                        blocks.push_back(std::move(B));
                        filling.push_back(1);
                    } else {
                        b = it->second;
                        filling.push_back(0);
                        if (blocks[b].rowptr[l] != 0)   // the block has entries in rows this occurrence lacks
                            throw Error(AIM_E_ARG, "near field not repetition-compressible (element " +
                                                       std::to_string(e) + ")");
                    }
                    fs.push_back(f);
                    bs.push_back(b);
                    cursor.push_back(0);
                }
                Block& B = blocks[bs[k]];
                if (filling[k]) {
                    B.col.push_back(loc[n]);
                    B.src.push_back(t);
                } else {
                    // the occurrence must have its block's structure
                    const int64_t c = B.rowptr[l] + cursor[k]++;
                    if (B.rowptr[l] < 0 || c >= B.rowptr[l + 1] || B.col[c] != loc[n])
                        throw Error(AIM_E_ARG, "near field not repetition-compressible (element " +
                                                   std::to_string(e) + ", row " + std::to_string(l) + ")");
                }
            }
            // close row l of the blocks being filled; check row lengths of the others
            for (size_t k = 0; k < fs.size(); ++k) {
                Block& B = blocks[bs[k]];
                if (filling[k]) {
                    B.rowptr[l + 1] = (int64_t)B.col.size();
                } else {
                    if (B.rowptr[l] + cursor[k] != B.rowptr[l + 1])
                        throw Error(AIM_E_ARG, "near field not repetition-compressible (row length)");
                    cursor[k] = 0;
                }
            }
        }
        // blocks first seen after row 0 have unset row pointers before their
        // first row: fill forward (empty rows)
        for (size_t k = 0; k < fs.size(); ++k)
            if (filling[k]) {
                Block& B = blocks[bs[k]];
                for (int l = 0; l < ne_rows; ++l)
                    if (B.rowptr[l + 1] < 0) B.rowptr[l + 1] = B.rowptr[l];
            }
        for (size_t k = 0; k < fs.size(); ++k) {
            slot_f.push_back(fs[k]);
            slot_b.push_back(bs[k]);
        }
        slot_ptr[e + 1] = (int64_t)slot_f.size();
    }
    // concatenate the dictionary
    std::vector<int64_t> brow(blocks.size()), rowptr, src;
    std::vector<int32_t> col;
    for (size_t b = 0; b < blocks.size(); ++b) {
        brow[b] = (int64_t)rowptr.size();
        const int64_t o = (int64_t)col.size();
        for (int64_t v : blocks[b].rowptr) rowptr.push_back(o + v);
        col.insert(col.end(), blocks[b].col.begin(), blocks[b].col.end());
        src.insert(src.end(), blocks[b].src.begin(), blocks[b].src.end());
    }
    bool contig = true;
    for (int e = 0; e < ne && contig; ++e)
        for (int64_t q = rptr[e]; q < rptr[e + 1]; ++q)
            if (rows[q] != rows[rptr[e]] + (q - rptr[e])) {
                contig = false;
                break;
            }
    auto up32 = [&](const std::vector<int32_t>& v) {
        int32_t* d = p->alloc<int32_t>(std::max<size_t>(1, v.size()));
        if (!v.empty()) h2d(d, v.data(), sizeof(int32_t) * v.size(), s);
        return d;
    };
    auto up64 = [&](const std::vector<int64_t>& v) {
        int64_t* d = p->alloc<int64_t>(std::max<size_t>(1, v.size()));
        if (!v.empty()) h2d(d, v.data(), sizeof(int64_t) * v.size(), s);
        return d;
    };
    p->cz_el_of = up32(el_of);
    p->cz_loc = up32(loc);
    p->cz_slot_ptr = up64(slot_ptr);
    p->cz_slot_f = up32(slot_f);
    p->cz_slot_b = up32(slot_b);
    p->cz_brow = up64(brow);
    p->cz_brow_h = brow;
    p->cz_rowptr = up64(rowptr);
    p->cz_col = up32(col);
    p->cz_val = p->alloc<double2>(std::max<size_t>(1, src.size()));
    if (!src.empty()) {
        int64_t* d_src = up64(src);
        cz_gather_kernel<<<(unsigned)((src.size() + 255) / 256), 256, 0, s>>>(p->nval, d_src, (long long)src.size(),
                                                                             p->cz_val);
        note_launch("cz_gather");
        AIM_CUDA(cudaStreamSynchronize(s));
        p->release(d_src);
    }
    p->cz_contig = contig ? 1 : 0;
    p->cz_max_slots = 0;
    for (int e = 0; e < ne; ++e) p->cz_max_slots = std::max<int>(p->cz_max_slots, (int)(slot_ptr[e + 1] - slot_ptr[e]));
    p->cmp_nnz = (int64_t)col.size();
    p->cmp_blocks = (int64_t)blocks.size();
    // single group, contiguous elements: the SpMM form (pairs of every block)
    p->cz_spmm = 0;
    if (contig && ng == 1 && getenv("AIM_CZ_SPMM") == nullptr) {
        std::vector<std::vector<int32_t>> pe(blocks.size()), pf(blocks.size());
        for (int e = 0; e < ne; ++e)
            for (int64_t sl = slot_ptr[e]; sl < slot_ptr[e + 1]; ++sl) {
                pe[slot_b[sl]].push_back(e);
                pf[slot_b[sl]].push_back(slot_f[sl]);
            }
        std::vector<int32_t> ape, apf, first(ne);
        p->cz_pairs.clear();
        for (size_t b = 0; b < blocks.size(); ++b) {
            p->cz_pairs.push_back({(int64_t)ape.size(), (int64_t)pe[b].size()});
            ape.insert(ape.end(), pe[b].begin(), pe[b].end());
            apf.insert(apf.end(), pf[b].begin(), pf[b].end());
        }
        for (int e = 0; e < ne; ++e) first[e] = rows[rptr[e]];
        p->cz_pe = up32(ape);
        p->cz_pf = up32(apf);
        p->cz_first = up32(first);
        p->cz_n = (int)(rptr[1] - rptr[0]);
        p->cz_xt = p->alloc<double2>((size_t)p->cz_n * ne);
        p->cz_yt = p->alloc<double2>((size_t)p->cz_n * ne);
        p->cz_spmm = 1;
    }
    std::vector<int32_t> rep(ng, -1);
    for (int e = 0; e < ne; ++e)
        if (rep[grp[e]] < 0) rep[grp[e]] = e;
    build_compressed_pi(p, grp, rep, base, s);
    p->cmp_on = 1;
}

void launch_near_cmp(aim_plan* p, const void* x, void* y, int R, cudaStream_t s) {
    const unsigned grid = (unsigned)((p->N * 32 + 255) / 256);
    if (R == 1 && p->cz_spmm) {
        const int n = p->cz_n, ne = p->el_count;
        const long long tot = (long long)n * ne;
        const unsigned gt = (unsigned)((tot + 255) / 256);
        cz_transpose_kernel<<<gt, 256, 0, s>>>((const double2*)x, n, ne, n, p->cz_first, p->cz_xt, 1);
        note_launch("cz_transpose");
        AIM_CUDA(cudaMemsetAsync(p->cz_yt, 0, sizeof(double2) * tot, s));
        for (size_t b = 0; b < p->cz_pairs.size(); ++b) {
            const int m = (int)p->cz_pairs[b].second;
            if (!m) continue;
            // block b's row pointers: brow is on the device; the host copy is kept
            const dim3 g2((unsigned)((n + kSpRows - 1) / kSpRows), (unsigned)((m + kSpPairs - 1) / kSpPairs));
            near_spmm_kernel<<<g2, 256, 0, s>>>(p->cz_rowptr + p->cz_brow_h[b], p->cz_col, p->cz_val,
                                                p->cz_pe + p->cz_pairs[b].first, p->cz_pf + p->cz_pairs[b].first, m, n,
                                                ne, p->cz_xt, p->cz_yt);
            note_launch("near_spmm");
        }
        cz_transpose_kernel<<<gt, 256, 0, s>>>((const double2*)y, n, ne, n, p->cz_first, p->cz_yt, 0);
        note_launch("cz_transpose");
        return;
    }
    if (R == 1 && p->cz_contig && p->cz_max_slots <= kCzMaxSlots) {
        near_cmp1_kernel<<<grid, 256, 0, s>>>(p->el_rows, p->el_rptr, p->cz_el_of, p->cz_loc, p->cz_slot_ptr,
                                              p->cz_slot_f, p->cz_slot_b, p->cz_brow, p->cz_rowptr, p->cz_col,
                                              p->cz_val, (const double2*)x, p->N, (double2*)y);
        note_launch("near_cmp1");
        return;
    }
    near_cmp_kernel<double2><<<grid, 256, 0, s>>>(p->el_rows, p->el_rptr, p->cz_el_of, p->cz_loc, p->cz_slot_ptr,
                                                  p->cz_slot_f, p->cz_slot_b, p->cz_brow, p->cz_rowptr, p->cz_col,
                                                  p->cz_val, p->cz_contig, (const double2*)x, p->N, R, (double2*)y);
    note_launch("near_cmp");
}

}  // namespace aim
