/*
 * aim.h -- C ABI of the B200-native AIM-accelerated EFIE matvec / GMRES
 * (hot path of Patel, Triverio, Hum, arXiv 1712.02443, §V "Acceleration with
 * AIM"; operator readings D1-D17 in SURVEY.md §8(c) and
 * DESIGN.md).
 *
 * The operator (eq. Gouter1, reading D1):
 *
 *   Z_eq = Z_corr + j k eta0 ( sum_{psi=x,y,z} P_psi^T H P_psi - k^-2 P_phi^T H P_phi )
 *
 *   P_psi   projection onto an AIM grid of spacing h, stencil order M,
 *           (M+1)^3 nodes per RWG (step (i); D2, D3, D4)
 *   H       Toeplitz convolution with G(R) = exp(-jkR)/(4 pi R), G(0) = 0
 *           (step (ii), eq. AIM_step2; D6, D11, D12)
 *   P^T     interpolation (step (iii))
 *   Z_corr  near-field precorrection on pairs ||c_m - c_n|| <= near_radius
 *           (D5, D8, D9)
 *
 * Conventions for every entry point:
 *   - Complex numbers are interleaved (re, im) float64 pairs (complex128).
 *   - Vectors x, y, V, J have layout [N][nrhs] with the RHS index fastest.
 *   - "device" pointers are CUDA device pointers on the device that was
 *     current when the plan was created; "host" pointers are ordinary host
 *     memory (pinned or pageable).
 *   - The caller owns every buffer it passes.  The library never frees them
 *     and keeps no pointer to them after the call returns.  The plan owns all
 *     device memory it allocates until aim_plan_destroy().
 *   - Streams are passed as `void*` holding a cudaStream_t (NULL = legacy
 *     default stream).  Stream-ordered entry points are asynchronous.
 *   - Every function returns an aim_status.  On a negative status a
 *     thread-local message is available from aim_last_error(); outputs are
 *     unspecified.  AIM_NOT_CONVERGED (=1) is a flag, not an error.
 *   - No entry point falls back to a CPU implementation: if the CUDA device
 *     or a kernel launch fails the call returns AIM_E_CUDA.
 */
#ifndef AIM_H
#define AIM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct aim_plan aim_plan; /* opaque */

typedef enum aim_status {
    AIM_OK = 0,
    AIM_NOT_CONVERGED = 1, /* aim_gmres: tolerance not reached in max_iters   */
    AIM_E_ARG = -1,        /* bad scalar argument / NULL pointer / nrhs < 1    */
    AIM_E_MESH = -2,       /* mesh topology error                 */
    AIM_E_GRID = -3,       /* grid or index space exceeds 32-bit addressing    */
    AIM_E_NOMEM = -4,      /* device allocation failed                         */
    AIM_E_CUDA = -5,       /* CUDA runtime / launch error                      */
    AIM_E_NCCL = -6,       /* NCCL failure (slab-decomposed multi-GPU path)     */
    AIM_E_BREAKDOWN = -7   /* aim_gmres: a non-finite value (NaN/Inf) in the
                              right-hand side, an Arnoldi coefficient, the
                              Hessenberg solve or the residual; J unspecified  */
} aim_status;

enum { AIM_C128 = 0, AIM_C64 = 1 };

typedef struct aim_info {
    int64_t n_rwg;          /* N                                                */
    int64_t n_tri;
    int32_t M;              /* stencil order (BASELINE.json's "order M")        */
    int32_t S;              /* (M+1)^3 nodes per stencil                        */
    int32_t grid_origin[3]; /* lattice index of grid node (0,0,0)  (D4)         */
    int32_t grid_dims[3];   /* Nx, Ny, Nz (unpadded grid)                       */
    int32_t fft_dims[3];    /* Px, Py, Pz >= 2 Na - 1 (D11)                     */
    int64_t n_nodes;        /* Nx Ny Nz                                         */
    int64_t nnz_proj;       /* N S projection entries                           */
    int64_t nnz_near;       /* near-field (precorrected) entries                */
    double k, h, near_radius;
    int64_t device_bytes;   /* device memory owned by the plan (workspaces incl.) */
    double plan_seconds;    /* wall time of aim_plan_create                     */
    int32_t conv_mode;      /* 0: 3-D FFT convolution, spectrum octant
                               [(Px/2+1)][(Py/2+1)][(Pz/2+1)];
                               1: planar -- 2-D FFT in x,y and direct Toeplitz
                               product in z, spectrum [(Px/2+1)][(Py/2+1)][Nz],
                               y passes and z product fused in one kernel;
                               2: planar with separate y passes and a z
                               Toeplitz kernel (same spectrum; grids whose
                               Py x Nz plane does not fit shared memory)      */
    int32_t precision;      /* AIM_C128 or AIM_C64                               */
} aim_info;

/*
 * aim_plan_create -- build the AIM operator for a closed triangle mesh.
 *
 * vertices   host  float64 [nv][3]   vertex coordinates (lambda = 1 units)
 * triangles  host  int32   [nt][3]   vertex indices
 * rwg_edges  host  int32   [N][4]    {va, vb, t_plus, t_minus}: the RWG on the
 *            edge (va, vb) shared by triangles t_plus and t_minus; current
 *            flows from t_plus into t_minus:
 *              Lambda = l/(2A+) (r - p+) on t+,  l/(2A-) (p- - r) on t-
 *            ("RWG basis function").
 * k          wavenumber > 0 (k = 2 pi for lambda = 1)
 * h          AIM grid spacing > 0 (lattice h Z^3 anchored at the origin, D4)
 * M          stencil order in [1, 6] ("N_O")
 * near_radius  >= 0; pairs with ||c_m - c_n|| <= near_radius (1 + 1e-9) are
 *            treated exactly (D5)
 * precision  AIM_C128, or AIM_C64 (BASELINE.json configs[4]; reading D16): the
 *            plan is computed in fp64 and its tables (weights, near values,
 *            spectrum, twiddles) rounded once to fp32 / complex64; the matvec
 *            then reads and writes complex64 vectors and runs the FFT and
 *            all accumulation in fp32.  aim_gmres / aim_planewave_rhs need an
 *            AIM_C128 plan (AIM_E_ARG otherwise).
 * dist       must be NULL (single-GPU plan); the slab-decomposed multi-GPU
 *            operator is aim_slab_create below
 * out        receives the plan
 *
 * Errors: AIM_E_ARG (k <= 0, h <= 0, M outside [1,6], near_radius < 0,
 * NULL pointers, N < 1), AIM_E_MESH (index out of range, t+ == t-, triangle
 * not containing va and vb, zero-area triangle), AIM_E_GRID (padded grid
 * > 2^31 points or nnz > 2^31 - 1), AIM_E_NOMEM, AIM_E_CUDA.
 * Synchronous.  Uses the current CUDA device.
 */
int aim_plan_create(const double* vertices, int64_t nv,
                    const int32_t* triangles, int64_t nt,
                    const int32_t* rwg_edges, int64_t n_rwg,
                    double k, double h, int32_t M, double near_radius,
                    int32_t precision, const void* dist, aim_plan** out);

/* Release every device buffer of the plan.  NULL is accepted. */
int aim_plan_destroy(aim_plan* plan);

/* Fill *info.  Host call, no device work. */
int aim_plan_info(const aim_plan* plan, aim_info* info);

/*
 * aim_matvec -- y := Z_eq x for nrhs right-hand sides (PAPER.md:539-559,
 * steps (i)-(iii) plus the precorrected near field).
 * x, y: device complex128 [N][nrhs] (complex64 for an AIM_C64 plan), must not
 * overlap.  nrhs >= 1.
 * Stream-ordered on `stream`; workspaces for this nrhs are allocated on the
 * first call (synchronously) and reused afterwards.
 */
int aim_matvec(aim_plan* plan, const void* x, void* y, int32_t nrhs, void* stream);

/*
 * aim_matvec_host -- the same product with HOST buffers: copies x to the
 * device, runs aim_matvec, copies y back, and synchronises (end-to-end path).
 */
int aim_matvec_host(aim_plan* plan, const void* x_host, void* y_host, int32_t nrhs);

/*
 * aim_matvec_host_steps -- `nsteps` products y_i := Z_eq x_i from HOST buffers
 * with the copies overlapped (end-to-end path for a stream of inputs): step
 * i's host->device copy, step i-1's product and step i-2's device->host copy
 * run concurrently on three streams (two device slots per direction, ordered
 * by events).  xs[i], ys[i]: host pointers to [N][nrhs] complex128
 * (complex64 for AIM_C64 plans); page-locked memory is needed for the copies
 * to overlap (pageable memory works, serialised).  xs[i] may repeat a
 * pointer; ys[i] must not alias another ys[j] written concurrently (j = i+-1).
 * Synchronous: returns when every y_i is in host memory.
 */
int aim_matvec_host_steps(aim_plan* plan, const void* const* xs, void* const* ys, int32_t nsteps,
                          int32_t nrhs);

/*
 * aim_gmres -- solve Z_eq J = V by restarted GMRES(restart) from J0 = 0
 * (reading D15: CGS2 Arnoldi, complex Givens rotations,
 * stop when ||V - Z J|| / ||V|| <= tol, the true residual being recomputed
 * at the end of each cycle).
 * V, J: device complex128 [N].  max_iters <= 0 means 20000.
 * fixed_iters > 0 runs exactly that many inner iterations and returns the
 * iterate (parity protocol "at equal iteration counts"); 0 = off.
 * iters, rel_res: host outputs (may be NULL).  Synchronous.
 * Returns AIM_OK, or AIM_NOT_CONVERGED with J = the last iterate.
 */
int aim_gmres(aim_plan* plan, const void* V, void* J, int32_t restart, double tol,
              int32_t max_iters, int32_t fixed_iters, int32_t* iters, double* rel_res);

/*
 * aim_gmres_history -- the residual estimates |g_{j+1}| / ||V|| of every
 * inner iteration of the last aim_gmres / aim_slab_gmres on this plan (D15),
 * in order.  out: host float64 [cap] (may be NULL when cap == 0); *count
 * receives the number of iterations (copies min(count, cap) values).  Host.
 */
int aim_gmres_history(const aim_plan* plan, double* out, int32_t cap, int32_t* count);

/* ---- block-Jacobi preconditioner -------------- */
/* The paper preconditions GMRES ("GMRES with an ILU-2 preconditioner",
 * PAPER.md:682, §VI-A); SPEC.md:493-501 substitutes per-element dense block
 * solves, which this library builds (reading D18):
 *   M = blockdiag_e Z_ex_sym[e, e],
 * e the connected surfaces of the mesh (the array elements' equivalent
 * surfaces), Z_ex_sym the exact symmetrised Galerkin entries (D8, D9) over
 * ALL RWG pairs of the element.  Elements that are translates of each other
 * (same local topology, corners equal to 1e-9 of the element size) share one
 * block ("only need to be calculated once for each distinct element",
 * PAPER.md:422-425).  Blocks are inverted on the device (Gauss-Jordan with
 * partial pivoting).  Once built, aim_gmres solves Z M^-1 u = V, J = M^-1 u
 * (right preconditioning; residuals and tolerance refer to Z J = V). */
enum { AIM_PRECOND_NONE = 0, AIM_PRECOND_BLOCK_JACOBI = 1 };
/* Build (kind 1) or remove (kind 0) the preconditioner.  Synchronous.
 * Errors: AIM_E_ARG (AIM_C64 plan, unknown kind), AIM_E_NOMEM,
 * AIM_E_BREAKDOWN (a singular or non-finite block; nothing is kept). */
int aim_precond_build(aim_plan* plan, int32_t kind);
/* y := M^-1 x, device complex128 [N], no overlap.  Stream-ordered.
 * AIM_E_ARG if no preconditioner is built. */
int aim_precond_apply(aim_plan* plan, const void* x, void* y, void* stream);
/* Host: out[5] = {built (0/1), elements, distinct blocks, largest block,
 * bytes of the inverses}. */
int aim_precond_info(const aim_plan* plan, int64_t* out);

/* ---- repetition-compressed operators (NEXT-3) -------------------------- */
/*
 * aim_plan_compress -- mode 1: build and use a repetition-compressed copy of
 * the precorrected near field ("matrices ... only need to be calculated once
 * for each distinct element").  Elements (connected
 * surfaces) that are translates of each other by integer multiples of h sit
 * identically on the grid, so the near block between elements e and f depends
 * only on (group(e), group(f), lattice offset f - e): one dictionary block per
 * key, plus per element its neighbour elements and their keys.  Every
 * occurrence's structure is verified equal to its block's; the values are
 * those of the key's first occurrence (other occurrences differ by rounding
 * only).  aim_matvec then reads the dictionary instead of the near CSR.
 * The same translation fixes the projection weights (D2 weights depend only
 * on positions relative to the stencil base): when the representatives'
 * (local row, stencil node) pairs number at most half the projection CSR,
 * single-RHS products project through one node-sorted template per group
 * (over the box of the representative's stencil nodes, summed over the
 * elements whose box holds the node, in ascending element order) and
 * interpolate with the representative's weight row; products with nrhs > 1
 * keep the general projection/interpolation tables.
 * mode 0: back to the general tables.  Synchronous.  Errors: AIM_E_ARG
 * (AIM_C64 plan; a structure mismatch -- the plan is left uncompressed).
 */
int aim_plan_compress(aim_plan* plan, int32_t mode);
/* Host: out[6] = {compressed (0/1), dictionary blocks, dictionary entries,
 * near entries of the general CSR, projection/interpolation compressed (0/1),
 * projection template entries}. */
int aim_compress_info(const aim_plan* plan, int64_t* out);

/* ---- array elements and the reduced (macromodel) system (NEXT-2) -------- */
/*
 * aim_plan_elements -- the array elements as the library enumerates them: the
 * connected surfaces of the mesh (triangles joined by an RWG), ordered by
 * their smallest RWG id; within an element the RWGs are in ascending id.
 * elem_of_rwg: host int32 [N] (or NULL) element of every RWG; group: host
 * int32 [n_elements] (or NULL) translate group of every element (elements
 * that are translates of one another share a group, D18); *n_elements.
 */
int aim_plan_elements(aim_plan* plan, int32_t* elem_of_rwg, int32_t* group, int32_t* n_elements);

/*
 * aim_reduced_set -- the macromodel blocks of the reduced system
 *   ( D - G^(E^,J^) T A^-1 B ) E^ = V^        (eq. finalsystem)
 * per element TYPE d (n_types types; "only need to be calculated once for each
 * distinct element").  Host complex128 row-major arrays,
 * the blocks of all types concatenated in type order:
 *   D  [nhat_d][nhat_d]
 *   T  [nhat_d][nint_d]   transfer matrix (eq. Tm1)
 *   A  [nint_d][nint_d]   interior operator A_m (eq. JM)
 *   B  [nint_d][nhat_d]   B_m (eq. JM)
 * nhat_d = RWGs of an element of type d on its equivalent surface (rows in
 * ascending RWG id, see aim_plan_elements), nint_d = interior unknowns.
 * elem_type: host int32 [n_elements], the type of every element.  The library
 * copies the blocks, inverts every A_d on the device and keeps D_d and
 * K_d = T_d A_d^-1 B_d.  Synchronous.  Errors: AIM_E_ARG (sizes or element
 * count not matching the mesh, AIM_C64 plan), AIM_E_NOMEM, AIM_E_BREAKDOWN
 * (singular A_d).
 */
int aim_reduced_set(aim_plan* plan, int32_t n_types, const int32_t* nhat, const int32_t* nint, const void* D,
                    const void* T, const void* A, const void* B, const int32_t* elem_type, int32_t n_elements);
/*
 * aim_reduced_matvec -- out := (D - G T A^-1 B) Y (eq. MV_product1,
 * PAPER.md:512-523) with G the AIM exterior operator; with the sign
 * convention of reading D1, G = -Z_eq, so out = D Y + Z_eq (K Y).  Y, out:
 * device complex128 [N], no overlap.  Stream-ordered.
 */
int aim_reduced_matvec(aim_plan* plan, const void* Y, void* out, void* stream);
/* GMRES on the reduced system (D15), as aim_gmres with the
 * operator of aim_reduced_matvec (no preconditioner).  Synchronous. */
int aim_reduced_gmres(aim_plan* plan, const void* V, void* E, int32_t restart, double tol, int32_t max_iters,
                      int32_t fixed_iters, int32_t* iters, double* rel_res);

/*
 * aim_planewave_rhs --V_m = <Lambda_m, E_inc>, E_inc(r) = E0 pol exp(-j k khat.r)
 * (PAPER.md:455-459 with the sign convention of D1; D14), 7-point rule.
 * khat, pol: host float64[3]; V: device complex128 [N].  Stream-ordered.
 */
int aim_planewave_rhs(aim_plan* plan, const double* khat, const double* pol,
                      double E0_re, double E0_im, void* V, void* stream);

/* ---- stage entry points (composition and per-stage parity) -------------- */
/* Grid arrays have layout [4][Nx][Ny][Nz][nrhs], components (x, y, z, phi). */

/* Q := P x   (step (i)).  x device [N][nrhs]. */
int aim_project(aim_plan* plan, const void* x, void* Q, int32_t nrhs, void* stream);

/* Phi := H Q (step (ii)), zero-padded FFT convolution.  Q is not modified;
 * Q and Phi may alias. */
int aim_convolve(aim_plan* plan, const void* Q, void* Phi, int32_t nrhs, void* stream);

/* y := j k eta0 [sum_xyz P^T Phi - k^-2 P_phi^T Phi_phi] (step (iii))
 *      + (add_near ? Z_corr x : 0).   With Phi == NULL only the near part. */
int aim_interpolate(aim_plan* plan, const void* Phi, const void* x, void* y,
                    int32_t nrhs, int32_t add_near, void* stream);

/* ---- plan export (host copies, for parity tests) ------------------------ */
enum {
    AIM_EXPORT_BASES = 0,      /* int32   [N][3]   absolute stencil base s_n     */
    AIM_EXPORT_WEIGHTS = 1,    /* float64 [N][S][4] projection weights          */
    AIM_EXPORT_NEAR_ROWPTR = 2,/* int64   [N+1]                                 */
    AIM_EXPORT_NEAR_COL = 3,   /* int32   [nnz_near] (ascending within a row)   */
    AIM_EXPORT_NEAR_VAL = 4,   /* complex128 [nnz_near] Z_corr                  */
    AIM_EXPORT_GREEN = 5,      /* complex128 spectrum, shape per aim_info.conv_mode */
    AIM_EXPORT_PROJ_ROWPTR = 6,/* int32   [Nx Ny Nz + 1]                        */
    AIM_EXPORT_PROJ_ENT = 7    /* int32   [N S] entries n*S + u                  */
};
/* Copy table `what` into host memory `dst` of `bytes` bytes (must be exact). */
int aim_plan_export(const aim_plan* plan, int32_t what, void* dst, int64_t bytes);

/* ---- live stage timing (bench accounting) ------------------------------- */
/* Stage ids of one aim_matvec (all on the caller's stream; launch order:
 * NEAR, PROJECT, FFT_X, FFT_YZ, IFFT_X, INTERP). */
enum {
    AIM_STAGE_PROJECT = 0,   /* H1 projection gather                                 */
    AIM_STAGE_FFT_X = 1,     /* H2 x forward pass, zero-pad fused                    */
    AIM_STAGE_FFT_YZ = 2,    /* H2-H4 y fwd, z convolution x spectrum, y inv         */
    AIM_STAGE_IFFT_X = 3,    /* H4 x inverse pass, pruned                            */
    AIM_STAGE_NEAR_WAIT = 4, /* (unused: 0)                                          */
    AIM_STAGE_INTERP = 5,    /* H5 interpolation, adds the far field to y            */
    AIM_STAGE_NEAR = 6,      /* H6 near-field SpMV, writes y                         */
    AIM_NUM_STAGES = 7
};
/* enable != 0: every subsequent aim_matvec records CUDA events around each
 * stage on its stream; enable == 0 stops and discards.  Host call. */
int aim_profile(aim_plan* plan, int32_t enable);
/* Synchronise on the recorded events and write the summed milliseconds per
 * stage into ms[AIM_NUM_STAGES] and the number of profiled matvecs into *count;
 * resets the accumulators. */
int aim_profile_read(aim_plan* plan, double* ms, int64_t* count);

/* ---- slab-decomposed multi-GPU product ---------------- */
/* BASELINE.json north_star: "the grid is slab-decomposed along x, the 3D FFT
 * transposes run as NCCL all-to-all over NVLink, basis functions and
 * precorrection rows are partitioned by owning slab with stencil halos".
 * The unpadded grid's x planes are cut into `world` contiguous slabs
 * [X[r], X[r+1]), balanced by the number of RWGs whose stencil base x index
 * (D3) lies in them, each at least M planes wide; rank r owns those RWGs
 * (near rows, weights) and the grid planes [X[r], X[r+1] + M).  Planar grids
 * (aim_info.conv_mode 1 or 2) and 3-D grids (conv_mode 0). */
typedef struct aim_slab aim_slab; /* opaque */

/* Host only (no device work): the partition of `world` slabs.
 * X: host int32 [world+1] plane bounds (0 = first grid plane, X[world] = Nx);
 * owner: host int32 [N] owning rank of each RWG, or NULL; grid_nx: host int32
 * (Nx), or NULL.  Errors: AIM_E_ARG (world * M > Nx, bad scalars),
 * AIM_E_MESH (index out of range). */
int aim_slab_partition(const double* vertices, int64_t nv, const int32_t* triangles, int64_t nt,
                       const int32_t* rwg_edges, int64_t n_rwg, double h, int32_t M, int32_t world,
                       int32_t* X, int32_t* owner, int32_t* grid_nx);

/* Fill `id` (host, `bytes` == NCCL_UNIQUE_ID_BYTES = 128) with a fresh NCCL
 * unique id (rank 0 calls this and broadcasts it).  libnccl.so.2 is loaded at
 * run time; AIM_E_NCCL if it cannot be. */
int aim_nccl_unique_id(void* id, int64_t bytes);

/*
 * aim_slab_create -- build the slab-decomposed operator (complex128).
 * Mesh and scalars as aim_plan_create.  Every rank passes the full mesh and
 * builds the grid, weights, projection and spectrum of the whole operator,
 * but near-field rows (the dominant plan time and memory) only for the RWGs
 * it owns; each rank keeps its own rows.  (With rank < 0 one base plan holds
 * every rank's near rows.)
 * rank in [0, world) with nccl_id (host, 128 bytes, the same on every rank):
 *   one process per GPU, exchanges over NCCL (grouped send/recv; halos to
 *   the neighbouring ranks, two all-to-all FFT transposes, a broadcast
 *   gather of y).  Collective: every rank must call it.
 * rank < 0 (nccl_id ignored): all `world` slabs on the current GPU in this
 *   process, exchanges as device copies with the same packing (checks the
 *   decomposition on one device).
 * Planar layouts whose y length has a compile-time plan (210, 784) store the y
 * pass's lines straight into the all-to-all blocks and load them back from
 * there (AIM_SLAB_FUSE_PACK=0: separate pack/unpack kernels, same bits).
 * Errors: as aim_plan_create; AIM_E_ARG also for world * M > Nx;
 * AIM_E_NCCL.  Synchronous.
 */
int aim_slab_create(const double* vertices, int64_t nv, const int32_t* triangles, int64_t nt,
                    const int32_t* rwg_edges, int64_t n_rwg, double k, double h, int32_t M,
                    double near_radius, int32_t world, int32_t rank, const void* nccl_id,
                    aim_slab** out);

/* y := Z_eq x, x and y device complex128 [N][nrhs] in the caller's RWG order,
 * replicated on every rank (x must be identical on every rank; every rank
 * receives all of y).  Stream-ordered on `stream`; with NCCL every rank must
 * call it (collective). */
int aim_slab_matvec(aim_slab* slab, const void* x, void* y, int32_t nrhs, void* stream);

/* aim_gmres on the slab-decomposed operator (D15).  V, J:
 * device complex128 [N], replicated on entry and exit.  Inside, every rank
 * keeps only its own rows [n0, n1) of the Krylov vectors; a product gathers
 * the input rows to every rank, and every dot product is a local partial sum
 * followed by an NCCL all-reduce of the (j+1) coefficients, so the iteration
 * is identical on every rank.  (rank < 0: the vectors span all rows, no
 * reduction.)  Collective with NCCL.  Synchronous.  Returns as aim_gmres. */
int aim_slab_gmres(aim_slab* slab, const void* V, void* J, int32_t restart, double tol,
                   int32_t max_iters, int32_t fixed_iters, int32_t* iters, double* rel_res);

/* Host: out[10] = {X[r], X[r+1], KY[r], KY[r+1] (owned ky range of the
 * x-pencil phase), n0, n1 (rank r's rows in the permuted order), local near
 * nnz (-1 if rank r is not held here), all-to-all bytes per RHS and matvec
 * (max over ranks, out + in), halo bytes per RHS and matvec, world}. */
int aim_slab_query(const aim_slab* slab, int32_t rank, int64_t* out);

/* Release everything (NCCL communicator included).  NULL is accepted. */
int aim_slab_destroy(aim_slab* slab);

/* Thread-local message for the last non-OK status ("" if none). */
const char* aim_last_error(void);

/* Number of kernel launches issued by this thread since the last reset
 * (bench accounting of "gpu_launches"). */
int64_t aim_launch_count(int32_t reset);

#ifdef __cplusplus
}
#endif
#endif /* AIM_H */
