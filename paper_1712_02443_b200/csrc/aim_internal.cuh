// Internal declarations of the AIM library (plan layout, launch helpers).
// See include/aim.h for the public contract and DESIGN.md for the design.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <functional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/aim.h"

namespace aim {

// ------------------------------------------------------------------ errors
struct Error : std::runtime_error {
    int status;
    Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};

#define AIM_CUDA(call)                                                                  \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess) {                                                        \
            throw ::aim::Error(e_ == cudaErrorMemoryAllocation ? AIM_E_NOMEM : AIM_E_CUDA, \
                               std::string(#call) + ": " + cudaGetErrorString(e_));      \
        }                                                                               \
    } while (0)

// Host -> device copy ordered on stream `s` and complete on return.  (A plain
// cudaMemcpy from pageable memory may return before its DMA has landed, and
// kernels on a non-blocking stream do not wait for the legacy stream.)
inline void h2d(void* d, const void* h, size_t bytes, cudaStream_t s) {
    AIM_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s));
    AIM_CUDA(cudaStreamSynchronize(s));
}

void note_launch(const char* name);  // counts launches, checks launch errors
long long launch_counter();          // kernels launched by this thread (aim_launch_count)
void add_launches(long long n);      // graph replays count their captured kernels
std::string& last_error();           // thread-local message behind aim_last_error()

inline int fail(int status, const std::string& msg) {
    last_error() = msg;
    return status;
}

// run an API body, mapping exceptions to aim_status codes
template <class F>
int guarded(F&& f) {
    try {
        last_error().clear();
        return f();
    } catch (const Error& e) {
        return fail(e.status, e.what());
    } catch (const std::bad_alloc&) {
        return fail(AIM_E_NOMEM, "host allocation failed");
    } catch (const std::exception& e) {
        return fail(AIM_E_CUDA, e.what());
    }
}

// eta0 = mu0 c with mu0 = 4 pi 1e-7 (reading D1; one fixed value).
constexpr double kPi = 3.14159265358979323846;
inline double eta0() { return 4.0e-7 * kPi * 299792458.0; }

// ------------------------------------------------------------ FFT pass plan
constexpr int kMaxStages = 12;

struct FftAxis {
    int P = 1;                       // transform length
    int nst = 0;                     // number of Stockham stages
    int radix[kMaxStages] = {0};     // radices, product == P
    unsigned long long nsM[kMaxStages] = {0};  // ceil(2^40 / Ns) of each stage (fast divide)
    int min_radix = 1;                          // smallest stage radix
    double2* tw = nullptr;           // device twiddles exp(-2 pi i e / P), e in [0,P)
    float2* tw32 = nullptr;          // the same rounded to complex64 (AIM_C64 plans)
};

// One batched 1-D pass over a tensor viewed as [outer][L][inner].
// Element type of the pass: prec 0 = complex128 (double2), 1 = complex64
// (float2); the data pointers are typed by it.
struct FftPass {
    const void* in;
    void* out;
    int prec = 0;
    long long outer;     // number of outer slices
    int Lin;             // input length along the axis (zero-padded to P)
    int Lout;            // output length along the axis (pruned from P)
    long long inner;     // element stride of the axis
    int TO, TI;          // tile: TO outer x TI inner lines per CTA
    int mode;            // 0 forward, 1 inverse, 2 turnaround (fwd, x spectrum, inv)
    FftAxis ax;
    // turnaround only: spectrum octant and the (kx, ky) decoding of `outer`
    const void* spec;
    int Px, Py;          // outer = (c Px + kx) Py + ky
    int PyH, PzH;        // octant extents Py/2+1, Pz/2+1
    // spec_mode 1 (x-line turnaround of the slab path): outer = c nky + kyl with
    // ky = off + kyl, inner = kz Rin + r, spectrum transposed [ay][az][ax]
    int spec_mode = 0;
    int Pz = 0, PxH = 0;
    int off = 0, nky = 1, Rin = 1;
    // Table-addressed lines (slab path: the all-to-all pack fused into the y-pass
    // store, the unpack into its load; compile-time plans only, modes 0/1,
    // complex128): element (oo, j, ii) of the output lives at
    // out + jout[j] + oo * inner + ii instead of out + (oo * Lout + j) * inner + ii,
    // the input likewise with jin.  Device tables of P entries, or null.
    const long long* jin = nullptr;
    const long long* jout = nullptr;
};

// Fused planar y/z pass (planar arrays): y fwd, direct z convolution with the
// 2-D spectrum G2[(Px/2+1)][(Py/2+1)][Nz], y inv; in place on [4][Px][Ny][Nz][R].
constexpr int kPlanarMaxNz = 16;
// The same kernel serves the slab-decomposed path with the roles of x and y
// swapped (outer = a local range of ky starting at `off`, lines along x).
struct PlanarPass {
    void* W;
    int prec = 0;        // as FftPass::prec
    int Px, Ny, Nz, R, RC;   // Px: number of outer planes per component in W
    int PyH;
    FftAxis ay;
    const void* spec;    // [(Pfold/2+1)][PyH][Nz]
    int off = 0;         // global index of outer plane 0
    int Pfold = 0;       // period of the outer axis (min-image fold of the spectrum index)
};

void launch_fft_pass(const FftPass& p, cudaStream_t s);
// Pass with jin/jout tables: false (nothing launched) if no compile-time plan takes it.
bool try_launch_fft_pass_tab(const FftPass& p, cudaStream_t s);
void launch_planar_yz(const PlanarPass& p, cudaStream_t s);
// z Toeplitz x G2 in place on lines [4][A][B][Nz][R]: (kx, ky) = (a, b) if kx_is_a
// else (b + 0, a + off) -- the second form serves the slab path's ky pencils
void launch_ztoeplitz(void* W, int prec, int A, int B, int Nz, int R, int kx_is_a, int off, int Px, int Py,
                      const void* spec, cudaStream_t s);
bool planar_supported(int Py, int Nz, int min_radix);
// fused mode-2 y/z pass (ymode2.cuh) for the compiled (Py, Nz) plans, one RHS,
// complex128; false if not applicable (the caller runs the separate passes)
bool launch_ymode2(void* W, int prec, int Px, int Ny, int Nz, int Py, int R, const void* spec, const FftAxis& ay,
                   cudaStream_t s);
void make_fft_axis(int P, FftAxis& ax);    // factorisation + device twiddles
int smooth_size_at_least(int n);           // smallest 2^a 3^b 5^c 7^d >= n

// Per-element dense blocks (block-Jacobi inverses, reduced-system D and K):
// element e uses block map[e] (n_d x n_d row-major at mats + off[d]).
// apply_blocks: out[rows_e] (+)= B_map[e] in[rows_e] for every element, as a
// GEMM over the elements sharing a block (jobs) or a GEMV per element.
struct PcJob {                    // block d shared by m elements listed at elist[eoff ..)
    int d, eoff, m, n;
    int64_t ioff;
};
struct BlockSet {
    int ndistinct = 0, maxn = 0;
    int64_t bytes = 0;
    double2* mats = nullptr;      // blocks, concatenated
    int64_t* off = nullptr;       // [ndistinct+1] (device)
    int32_t* map = nullptr;       // [elements] (device)
    std::vector<PcJob> jobs;
    int32_t* elist = nullptr;     // job element lists, then the GEMV elements
    int gemv_off = 0, gemv_cnt = 0;
};

// -------------------------------------------------------------------- plan
}  // namespace aim

struct aim_plan {
    int device = 0;
    int64_t N = 0, nt = 0, nv = 0;
    double k = 0, h = 0, r = 0;
    int M = 0, S = 0;
    int origin[3] = {0, 0, 0};
    int dims[3] = {0, 0, 0};     // Nx Ny Nz
    int pads[3] = {0, 0, 0};     // Px Py Pz
    int64_t Ng = 0;
    int64_t nnzP = 0, nnzN = 0;
    double plan_seconds = 0;

    // geometry (device)
    double* tri_qp = nullptr;     // [nt][7][3]
    double* tri_qw = nullptr;     // [nt][7]   weight x area
    double* tri_cor = nullptr;    // [nt][3][3]
    int32_t* tri_v = nullptr;     // [nt][3]
    int32_t* rwg_t = nullptr;     // [N][2]   t+, t-
    double* rwg_a = nullptr;      // [N][2]   alpha = +-l/(2A)
    double* rwg_p = nullptr;      // [N][2][3] free vertices
    double* rwg_c = nullptr;      // [N][3]   centre
    int32_t* base = nullptr;      // [N][3]   absolute stencil base
    int32_t* node0 = nullptr;     // [N]      grid index of the base node
    // host copies (element grouping of the preconditioner)
    std::vector<int32_t> h_tv;    // [nt][3] vertex ids
    std::vector<double> h_cor;    // [nt][3][3] corners
    std::vector<int32_t> h_rt;    // [N][2] t+, t-

    // operator tables (device)
    double* W = nullptr;          // [N][S][4] weights (x, y, z, phi)
    int32_t* prow = nullptr;      // [Ng+1]
    int32_t* pent = nullptr;      // [nnzP]  n*S + u
    int32_t* pn = nullptr;        // [nnzP]  n        (CSR order)
    double* Wc = nullptr;         // [nnzP][4] weights in CSR order (streamed by the projection)
    float* Wc32 = nullptr;        // [nnzP][4] complex64 plans
    int64_t* nrow = nullptr;      // [N+1]
    int32_t* ncol = nullptr;      // [nnzN]
    double2* nval = nullptr;      // [nnzN]
    // near rows to build (slab ranks: the owned RWGs); empty = every row
    std::vector<uint8_t> near_keep;
    int ncol_padded = 0;          // ncol/nval/nval32 padded >= 16 bytes past nnzN (bulk copies)
    // near rows in chunks of <= 1024 entries for the TMA-staged SpMV that runs
    // beside the FFT (k_near_stream.cu; built on first use)
    int ns_state = 0;             // 0 = not built, 1 = ready, -1 = not applicable
    int ns_count = 0;             // chunks
    int32_t* ns_crow = nullptr;   // [ns_count+1] first row of each chunk
    int64_t* ns_cent = nullptr;   // [ns_count+1] first entry of each chunk
    unsigned* ns_ctr = nullptr;   // chunk counter shared by the two launches
    // complex64 plans (reading D16): the fp64 tables rounded once
    int prec = AIM_C128;
    float* W32 = nullptr;         // [N][S][4]
    float2* nval32 = nullptr;     // [nnzN]
    float2* spec32 = nullptr;     // spectrum, as spec
    float2* nb_val32 = nullptr;   // [nbc][4]
    // near field in 4-row blocks (multi-RHS products; built on first use):
    // rows of a block are 4 consecutive RWGs in Morton order of their centres,
    // columns the sorted union of the 4 rows' columns, values dense 4 per column
    int64_t nb_count = 0;         // number of blocks (0 = not built)
    int64_t nbc = 0;              // block columns
    int32_t* nb_rows = nullptr;   // [nb_count][4] row ids, -1 = padding
    int64_t* nb_ptr = nullptr;    // [nb_count+1]
    int32_t* nb_col = nullptr;    // [nbc]
    double2* nb_val = nullptr;    // [nbc][4]
    // near field in 8- or 16-row blocks for the FP64 tensor-core SpMM (complex128,
    // R >= 8; built on first use): chunks of 4 union columns, a 32-bit
    // row x column presence mask per chunk, values packed (exactly nnzN)
    int64_t nm_count = 0;         // number of blocks (0 = not built)
    int64_t nm_chunks = 0;
    int nm_mt = 1;                // m-tiles per block (8 * nm_mt rows)
    int32_t* nm_rows = nullptr;   // [nm_count][8 nm_mt] row ids, -1 = padding
    int64_t* nm_cptr = nullptr;   // [nm_count+1] chunk ranges
    int64_t* nm_vptr = nullptr;   // [nm_count+1] packed value ranges
    uint32_t* nm_mask = nullptr;  // [nm_chunks][nm_mt]
    int32_t* nm_col = nullptr;    // [nm_chunks][4]
    double2* nm_val = nullptr;    // [nnzN]
    // interpolation in 8*im_mt-row blocks for the FP64 tensor cores (complex128,
    // R >= 8; built on first use): one chunk per union stencil node, k = component
    int64_t im_count = 0;         // number of blocks (0 = not built)
    int64_t im_chunks = 0;
    int im_mt = 2;
    int32_t* im_rows = nullptr;   // [im_count][8 im_mt]
    int64_t* im_cptr = nullptr;   // [im_count+1]
    int64_t* im_vptr = nullptr;   // [im_count+1] packed weight ranges (doubles)
    int32_t* im_node = nullptr;   // [im_chunks] grid node index
    uint32_t* im_mask = nullptr;  // [im_chunks][im_mt]
    double* im_val = nullptr;     // packed weights, phi scaled by -1/k^2
    int planar = 0;               // conv mode: 1 fused planar, 2 planar with separate passes (both
                                  // spec = G2, z by direct Toeplitz), 0 3-D FFT (spec = octant)
    double2* spec = nullptr;      // 3-D: [(Px/2+1)(Py/2+1)(Pz/2+1)]; planar: [(Px/2+1)(Py/2+1)][Nz]
    int64_t spec_len = 0;
    aim::FftAxis ax[3];

    // workspaces (device), sized for ws_nrhs
    int ws_nrhs = 0;
    double2* Q = nullptr;         // [4][Nx][Ny][Nz][R]   (also Phi)
    double2* W1 = nullptr;        // [4][Px][Ny][Nz][R]
    double2* W2 = nullptr;        // [4][Px][Py][Nz][R]
    // GMRES workspace (vectors of local length gm_n)
    int gm_restart = 0;
    long long gm_n = 0;
    double2* gm_V = nullptr;      // [(restart+1)][n]
    double2* gm_w = nullptr;      // [n]
    double2* gm_z = nullptr;      // [n] preconditioned vector (right preconditioning)
    double2* gm_part = nullptr;   // block partials + device coefficients
    double2* gm_host = nullptr;   // pinned host mirror of the coefficients
    cudaEvent_t gm_ev = nullptr;  // coefficients of the current iteration fetched
    std::vector<double> gm_hist;  // residual estimate |g_{j+1}|/||b|| of the last solve
    // array elements = connected surfaces of the mesh (built on first use by
    // ensure_elements): ordered by smallest RWG id, RWGs ascending within
    int el_count = 0;
    std::vector<int64_t> el_rptr_h;   // [el_count+1]
    std::vector<int32_t> el_rows_h;   // [N] RWG ids element-major
    std::vector<int32_t> el_group_h;  // [el_count] translate group (first element of the group defines it)
    std::vector<int32_t> el_reps_h;   // [groups] representative element of each group
    int32_t* el_rows = nullptr;   // device copies
    int64_t* el_rptr = nullptr;
    // repetition-compressed near field (aim_plan_compress, k_compress.cu)
    int cmp_on = 0, cz_contig = 0, cz_max_slots = 0;
    int64_t cmp_nnz = 0, cmp_blocks = 0;
    int32_t* cz_el_of = nullptr;  // [N] element of every RWG
    int32_t* cz_loc = nullptr;    // [N] local row of every RWG in its element
    int64_t* cz_slot_ptr = nullptr;   // [elements+1] neighbour slots
    int32_t* cz_slot_f = nullptr;     // [slots] neighbour element
    int32_t* cz_slot_b = nullptr;     // [slots] dictionary block
    int64_t* cz_brow = nullptr;   // [blocks] offset of the block's row pointers in cz_rowptr
    int64_t* cz_rowptr = nullptr; // concatenated block row pointers (absolute into cz_col / cz_val)
    int32_t* cz_col = nullptr;    // local column of the neighbour element
    double2* cz_val = nullptr;
    std::vector<int64_t> cz_brow_h;
    // single element group: sparse x dense form over the element pairs of each block
    int cz_spmm = 0, cz_n = 0;
    int32_t *cz_pe = nullptr, *cz_pf = nullptr, *cz_first = nullptr;   // pairs (e, f); first RWG of e
    std::vector<std::pair<int64_t, int64_t>> cz_pairs;               // per block: (offset, count) of its pairs
    double2 *cz_xt = nullptr, *cz_yt = nullptr;                      // [n][elements] transposed x, y
    // repetition-compressed projection / interpolation (single RHS): one
    // node-sorted template per group over the box of its representative's
    // stencil nodes, and per grid-node chunk (one CTA) the elements whose box
    // meets it; the interpolation reads the representative's weight row
    int cp_on = 0;
    int64_t cp_tpl_nnz = 0, cp_chunks = 0;
    int64_t* cp_cptr = nullptr;   // [chunks+1]
    int32_t* cp_cel = nullptr;    // elements meeting each chunk (ascending)
    int4* cp_ebox = nullptr;      // [elements] box corner (grid-relative) and group
    int4* cp_gdim = nullptr;      // [groups] box dims and offset of the group's template row pointers
    int32_t* cp_tptr = nullptr;   // concatenated template row pointers (absolute)
    int32_t* cp_tl = nullptr;     // template entry: local row of the element
    double* cp_tw = nullptr;      // template entry: [4] weights (x, y, z, phi)
    int32_t* cp_xfirst = nullptr; // [elements] first RWG (contiguous elements) or el_rptr
    int32_t* cp_wrow = nullptr;   // [N] RWG whose weight row the interpolation reads
    // element-batched projection: per group its elements, x transposed
    // Xt_d [n][ne_d] and the per-element box contributions Qt_d [nodes][ne_d][4]
    struct CpGroup {
        int ne, n, nodes, toff, eoff;
        int64_t xoff, qoff;
    };
    std::vector<CpGroup> cp_groups;
    int32_t* cp_gel = nullptr;      // group element lists, concatenated
    int64_t* cp_qbase = nullptr;    // [elements] offset of the element's Qt column (complex units)
    int32_t* cp_qstride = nullptr;  // [elements] stride between box nodes (4 ne_d)
    double2* cp_xt = nullptr;
    double2* cp_qt = nullptr;
    // block-Jacobi preconditioner (aim_precond_build): one dense inverse per
    // translate group
    int prec_on = 0;
    aim::BlockSet pc;
    // reduced (macromodel) system of PAPER.md eq. finalsystem (aim_reduced_set):
    // D and K = T A^-1 B per element type
    int rd_on = 0;
    aim::BlockSet rd_D, rd_K;
    double2* rd_t = nullptr;      // [N] K Y
    // host staging for aim_matvec_host
    int hs_nrhs = 0;
    double2* hx = nullptr;
    double2* hy = nullptr;

    // aim_matvec as CUDA graphs (k_matvec.cu matvec): one per (x, y, nrhs)
    struct MvGraph {
        const void* x;
        void* y;
        int R;
        cudaGraphExec_t exec;
        long long kernels;
    };
    std::vector<MvGraph> graphs;
    std::vector<char> mv_warm;    // an eager product has run for this nrhs
    cudaEvent_t gx_fork = nullptr, gx_join = nullptr;

    // aim_matvec_host_steps: double-buffered device vectors, copy streams, events
    int hp_nrhs = 0;
    double2* hp_x[2] = {nullptr, nullptr};
    double2* hp_y[2] = {nullptr, nullptr};
    cudaStream_t hp_in = nullptr, hp_out = nullptr;
    cudaEvent_t hp_ev_in[2] = {nullptr, nullptr}, hp_ev_mv[2] = {nullptr, nullptr}, hp_ev_out[2] = {nullptr, nullptr};

    // side stream for the near-field SpMV (overlaps the FFT passes)
    cudaStream_t side = nullptr;
    cudaEvent_t ev_x = nullptr, ev_n = nullptr;
    // high-priority stream for the FFT passes beside the near SpMV (AIM_NEAR_PRIO=1)
    cudaStream_t hi = nullptr;
    cudaEvent_t ev_h = nullptr;
    // live stage timing (aim_profile): kProfEvents events per profiled matvec
    int prof = 0;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    int64_t prof_count = 0;

    int64_t device_bytes = 0;
    std::vector<std::pair<void*, size_t>> allocs;
    cudaStream_t stream = nullptr;  // plan-private stream for synchronous calls

    template <class T>
    T* alloc(size_t count) {
        void* p = nullptr;
        if (count == 0) count = 1;
        cudaError_t e = cudaMalloc(&p, count * sizeof(T));
        if (e != cudaSuccess)
            throw aim::Error(AIM_E_NOMEM, std::string("cudaMalloc ") + std::to_string(count * sizeof(T)) +
                                              " bytes: " + cudaGetErrorString(e));
        allocs.emplace_back(p, count * sizeof(T));
        device_bytes += (int64_t)(count * sizeof(T));
        return (T*)p;
    }
    void release(void* p) {
        if (!p) return;
        for (size_t i = 0; i < allocs.size(); ++i)
            if (allocs[i].first == p) {
                device_bytes -= (int64_t)allocs[i].second;
                allocs.erase(allocs.begin() + i);
                break;
            }
        cudaFree(p);
    }
};

namespace aim {

constexpr int kProfEvents = 9;

// ---- whole-plan construction / teardown (aim_api.cu)
void create_plan(const double* V, int64_t nv, const int32_t* T, int64_t nt, const int32_t* E, int64_t N, double k,
                 double h, int M, double r, int prec, aim_plan* p);
void destroy_plan(aim_plan* p);

// ---- plan-building launches (k_plan.cu)
void build_weights(aim_plan* p, cudaStream_t s);
void build_projection_csr(aim_plan* p, const std::vector<int32_t>& node0_host, cudaStream_t s);
void build_near_list(aim_plan* p, cudaStream_t s);
void build_near_values(aim_plan* p, cudaStream_t s);
void build_green_spectrum(aim_plan* p, cudaStream_t s);
void build_near_blocks(aim_plan* p, cudaStream_t s);
// TMA-staged near SpMV overlapped with the FFT (k_near_stream.cu)
int near_overlap_mode();
int near_prio_mode();
int smem_carveout_max();
int near_overlap_ctas_per_sm();
bool near_stream_ready(aim_plan* p, cudaStream_t s);
void near_stream_reset(aim_plan* p, cudaStream_t s);
void launch_near_stream(aim_plan* p, const void* x, void* y, int ctas_per_sm, cudaStream_t s);
void build_near_mma(aim_plan* p, cudaStream_t s);
void build_interp_mma(aim_plan* p, cudaStream_t s);
void make_c64_blocks(aim_plan* p, cudaStream_t s);   // rounded nb_val for AIM_C64 plans

// ---- matvec launches (k_matvec.cu)
// x, y, Q, Phi are complex128 (double2) or complex64 (float2) by plan->prec
void launch_project(const aim_plan* p, const void* x, void* Q, int R, cudaStream_t s);
void launch_interp(aim_plan* p, const void* Phi, void* y, int R, bool accumulate, cudaStream_t s);
void launch_near(aim_plan* p, const void* x, void* y, int R, cudaStream_t s);
void launch_planewave(const aim_plan* p, const double* khat, const double* pol, double2 E0, double2* V,
                      cudaStream_t s);
void convolve(aim_plan* p, const void* Q, void* Phi, int R, cudaStream_t s);
void ensure_workspace(aim_plan* p, int R);
void matvec(aim_plan* p, const void* x, void* y, int R, cudaStream_t s);

// ---- GMRES (k_gmres.cu)
// Operator of a GMRES solve on vectors of local length n: matvec applies A,
// precond (optional) M^-1 (right preconditioning), allreduce (optional) sums a
// small device vector of complex values over the ranks (distributed Krylov
// vectors; stream-ordered).
struct GmresOps {
    long long n = 0;
    std::function<void(const double2*, double2*, cudaStream_t)> matvec;
    std::function<void(const double2*, double2*, cudaStream_t)> precond;
    std::function<void(double2*, int, cudaStream_t)> allreduce;
};
int gmres_core(aim_plan* p, const GmresOps& ops, const double2* b, double2* x, int restart, double tol,
               int max_iters, int fixed_iters, int* iters_out, double* rel_out);
int gmres(aim_plan* p, const double2* V, double2* J, int restart, double tol, int max_iters, int fixed_iters,
          int* iters, double* rel_res);

// ---- elements, per-element blocks, block-Jacobi preconditioner (k_precond.cu)
void ensure_elements(aim_plan* p, cudaStream_t s);
// finish a block set whose mats/off are filled: map, jobs, element lists
void setup_block_apply(aim_plan* p, BlockSet& b, const std::vector<int32_t>& map, const std::vector<int>& sizes,
                       cudaStream_t s);
void apply_blocks(aim_plan* p, const BlockSet& b, const double2* in, double2* out, bool accumulate, cudaStream_t s);
void free_blocks(aim_plan* p, BlockSet& b);
// batched Gauss-Jordan inversion in place of the blocks (n_d x n_d at mats + off_h[d]);
// throws AIM_E_BREAKDOWN on a singular block
void invert_blocks(double2* mats, const std::vector<int64_t>& off_h, const std::vector<int>& sizes, cudaStream_t s);
// C[m x n] = A[m x k] B[k x n], row-major complex128, device
void zgemm_rm(const double2* A, const double2* B, double2* C, int m, int n, int k, cudaStream_t s);
void build_precond(aim_plan* p, cudaStream_t s);
void apply_precond(aim_plan* p, const double2* in, double2* out, cudaStream_t s);
void free_precond(aim_plan* p);
// ---- repetition-compressed near field (k_compress.cu)
void build_compressed(aim_plan* p, cudaStream_t s);
void free_compressed(aim_plan* p);
void launch_near_cmp(aim_plan* p, const void* x, void* y, int R, cudaStream_t s);
void launch_project_cmp(const aim_plan* p, const void* x, void* Q, cudaStream_t s);   // cp_on, R = 1
// ---- reduced (macromodel) system (k_reduced.cu)
void reduced_set(aim_plan* p, int ntypes, const int32_t* nhat, const int32_t* nint, const double2* D,
                 const double2* T, const double2* A, const double2* B, const int32_t* elem_type, int nelem);
void reduced_matvec(aim_plan* p, const double2* Y, double2* out, cudaStream_t s);
void free_reduced(aim_plan* p);

}  // namespace aim
