/*
 * mrsolve_b200.h -- C ABI of the B200-native multi-RHS AMG-Krylov solve path.
 *
 * Plain C: pointers, sizes, int status codes; no torch or C++ types.  Built
 * into paper_2103_07329_b200/libmrsolve_b200.so (sm_100a).
 *
 * Two layers, mirroring the two boundaries of the reference package
 * (/root/reference/pkg/src/mrsolve):
 *
 *  1. Kernel plugin  -- replaces the `mrsolve.kernels` backend module
 *     (src/kernels/__init__.py:27-41, compiled twin src/kernels/_ckernels.pyx).
 *     Same operations, same arithmetic order, on DEVICE pointers, enqueued on
 *     a caller-supplied cudaStream_t (passed as void*).  Asynchronous.
 *
 *  2. Solver plan    -- replaces `solvers.prepare(config, A, team).run(B, X)`
 *     (src/solvers.py:850-959).  An opaque plan owns the uploaded AMG
 *     hierarchy (src/amg.py:199-239), the device workspaces and the captured
 *     CUDA graph of the whole solve; `mrs_plan_solve` runs one solve and
 *     returns SolveStats fields (src/solvers.py:80-92).
 *
 *  3. Native host setup -- the reference's Ruge-Stueben setup
 *     (src/amg.py:55-308) and eigenvalue-bound estimate (src/solvers.py:
 *     486-517), re-implemented in C++ with bitwise-identical output, so the
 *     uploaded hierarchy is the reference's.
 *
 * Conventions: vectors are (n, m) row-major float64 ("RHS-interleaved",
 * reference core.py:94-143).  Matrix values are float32 or float64
 * (val_bytes 4/8); column indices uint8/uint16/uint32 (idx_bytes 1/2/4).
 * Device CSR row pointers are int32 (nnz < 2^31); host CSR row pointers are
 * int64 like the reference's CsrBlock.
 */
#ifndef MRSOLVE_B200_H
#define MRSOLVE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
#define MRS_OK               0
#define MRS_ERR_ARG          1   /* bad shape / dtype / mode / alias          */
#define MRS_ERR_CUDA         2   /* CUDA runtime error                          */
#define MRS_ERR_UNSUPPORTED  3   /* configuration not on the device path        */
#define MRS_ERR_ALLOC        4   /* device or host allocation failed            */
#define MRS_ERR_BREAKDOWN    5   /* Krylov breakdown (column in stats)          */
#define MRS_ERR_SINGULAR     6   /* zero / missing diagonal                     */
#define MRS_ERR_DEGENERATE   7   /* AMG setup degeneracy after the retry        */
#define MRS_ERR_STATE        8   /* call out of order (e.g. solve before finalize) */
#define MRS_ERR_INSTABILITY  9   /* PBiCGStab recurrence drifted from the true residual */

/* csr_spmv accumulation modes (reference kernels/python_ref.py:24-27) */
#define MRS_MODE_ASSIGN 0   /* y  = A x     */
#define MRS_MODE_ADD    1   /* y += A x     */
#define MRS_MODE_SUB    2   /* y -= A x     */
#define MRS_MODE_RSUB   3   /* y  = b - A x */

/* Device CSR view.  All pointers are device pointers owned by the caller. */
typedef struct {
    int64_t nrows, ncols, nnz;
    const int32_t* row_ptr;   /* nrows + 1 */
    const void* col_idx;      /* nnz entries of idx_bytes */
    const void* values;       /* nnz entries of val_bytes */
    int32_t idx_bytes;        /* 1, 2 or 4 */
    int32_t val_bytes;        /* 4 or 8 */
    /* Slab-compressed 16-bit indices (optional, idx_bytes == 2): the column of
     * an entry in row i is slab_base[i >> slab_shift] + col_idx[k]. */
    const int32_t* slab_base; /* NULL: plain indices */
    int32_t slab_shift;
    int32_t pad_;
    /* Optional (NULL / 0: none): rows with more than long_thr entries, done by
     * whole CTAs instead of lane groups (same bits; the lane path skips them).
     * Device int32 array of n_long row indices. */
    const int32_t* long_rows;
    int32_t n_long;
    int32_t long_thr;
    /* Optional structure facts the caller knows from the host arrays (0 / -1:
     * unknown).  With them a single right-hand side product of a banded operator
     * runs on the TMA-fed "stream" kernel (csrc/stream.cu; same bits).
     *   band     max |column - row| over the entries, -1 unknown
     *   blk_max  most entries in any aligned block of 256 consecutive rows
     *   flags    bit 0: col_idx and values have >= 64 bytes of readable slack
     *            behind their nnz entries (stages are fetched in 16-byte units) */
    int32_t band;
    int32_t blk_max;
    int32_t flags;
    int32_t pad2_;
} mrs_csr;

/* Host CSR (the reference CsrBlock layout, core.py:146-254). */
typedef struct {
    int64_t nrows, ncols, nnz;
    const int64_t* row_ptr;
    const void* col_idx;
    const void* values;
    int32_t idx_bytes;
    int32_t val_bytes;
    const int32_t* slab_base; /* optional slab-relative 16-bit indices (see mrs_csr) */
    int32_t slab_shift;
    int32_t pad_;             /* flags.  bit 0: 32-bit columns may be compressed to
                               * slab-relative 16-bit ones by the upload, on the device
                               * (csrc/slab.cu; the rule of core.slab_compress) */
} mrs_host_csr;

/* ---- 1. kernel plugin (src/kernels/__init__.py:27-41) ------------------ */

/* _ckernels.pyx:30-57.  x: (A.ncols, m), y/b: (A.nrows, m).  b only for RSUB.
 * x must not alias y.  Per-(row, column) accumulation in CSR entry order with
 * separately rounded mul/add: bitwise equal to the reference kernel. */
int mrs_csr_spmv(const mrs_csr* A, const double* x, double* y, int64_t m,
                 int32_t mode, const double* b, void* stream);
/* Extension (no reference counterpart: its vectors are always float64): the same
 * product on float32 block vectors -- loads widened, float64 accumulation in entry
 * order, one rounding at the store.  m in {1, 2, 4, 8, 16, 32}; 16/32-bit columns;
 * 16-byte aligned vectors. */
int mrs_csr_spmv_f32(const mrs_csr* A, const float* x, float* y, int64_t m,
                     int32_t mode, const float* b, void* stream);
/* Diagnostics: launches of the single-RHS stream kernel (csrc/stream.cu) made by
 * this process so far -- lets tests and the bench see which path a product took. */
int64_t mrs_stream_launches(void);
/* Diagnostics: Galerkin products A_c = (R A) P that mrs_amg_setup ran on the GPU
 * (csrc/spgemm.cu; option "setup_gpu" / env MRS_SETUP_GPU=0 forces the host path). */
int64_t mrs_galerkin_gpu_count(void);

/* Vector kernels over (n, m) blocks; per-column scalars a, b, c are DEVICE
 * arrays of length m.  Same per-element expressions as _ckernels.pyx:82-162. */
int mrs_axpby(int64_t n, int64_t m, const double* a, const double* x,
              const double* b, double* y, void* stream);
int mrs_add2_scaled(int64_t n, int64_t m, double* y, const double* a,
                    const double* u, const double* b, const double* v, void* stream);
int mrs_fused_paired_update(int64_t n, int64_t m, double* y1, const double* a,
                            const double* u, const double* b, const double* s,
                            double* y2, const double* c, const double* w, void* stream);
/* Reductions write the full per-column result (m doubles, device) -- the
 * reduction over row blocks is done on the device in a fixed order, so the
 * result is deterministic (not the reference's sequential fold bitwise). */
int mrs_dot(int64_t n, int64_t m, const double* x, const double* y, double* out,
            void* stream);
int mrs_fused_update_dot(int64_t n, int64_t m, const double* a, const double* x,
                         const double* b, double* y, double* out, void* stream);
int mrs_fused_update_dot2(int64_t n, int64_t m, double* y, const double* u,
                          const double* c, const double* w, const double* z,
                          double* d1, double* d2, void* stream);

/* _ckernels.pyx:60-79 gs_sweep: one Gauss-Seidel half-sweep (forward != 0:
 * rows ascending) in place on x, v = b - c, v -= a_ik x_k for k != diag_pos[i]
 * in entry order, x_i = v / a_ii -- bitwise the sequential sweep (level
 * scheduled, sgs.cuh).  Square A; diag_pos int64[nrows] (device); b, c, x
 * (nrows, m) float64 device, m <= 256.  Synchronous on `stream` (the level
 * schedule is built on the host per call). */
int mrs_gs_sweep(const mrs_csr* A, const int64_t* diag_pos, const double* b,
                 const double* c, double* x, int64_t m, int32_t forward, void* stream);

/* ---- 2. solver plan (src/solvers.py:850-959) ---------------------------- */

#define MRS_METHOD_CG        0
#define MRS_METHOD_BICGSTAB  1   /* classical van der Vorst, solvers.py:219-293 */
#define MRS_METHOD_RBICGSTAB 2   /* reordered, two reduction groups, solvers.py:296-364 */
#define MRS_METHOD_PBICGSTAB 3   /* pipelined (op = A M, drift check), solvers.py:367-479 */
#define MRS_METHOD_STATIONARY 4  /* repeat one step of `precond` on X until the true residual
                                    meets rel_tol: MultiGrid (one V-cycle, multigrid_solve,
                                    solvers.py:683-710), Jacobi (one sweep, weight pc_weight) or
                                    Gauss-Seidel (one sweep, pc_direction) (_stationary_solve,
                                    solvers.py:962-978) */
#define MRS_METHOD_DIRECT    5   /* X = A^-1 B with the dense inverse given as the "coarse
                                    inverse" (n x n), precond NONE (direct_solve, :588-604) */

#define MRS_PC_NONE     0
#define MRS_PC_JACOBI   1        /* _SweepPrecond(jacobi), solvers.py:716-726,782-788 */
#define MRS_PC_MG       2        /* MultiGrid V-cycle, solvers.py:615-675 */
#define MRS_PC_SGS      3        /* _SweepPrecond(sgs_sweep), solvers.py:792-797 */
#define MRS_PC_CHEB     4        /* _SweepPrecond(chebyshev_apply), solvers.py:796-802: order in
                                    desc.pre.order, bounds = level 0 lmin/lmax */

#define MRS_SMOOTH_JACOBI     0  /* blas2.jacobi_sweep, blas2.py:165-185 */
#define MRS_SMOOTH_CHEBYSHEV  1  /* solvers.chebyshev_apply, solvers.py:520-571 */
#define MRS_SMOOTH_SGS        2  /* blas2.sgs_sweep (hybrid Gauss-Seidel, one leaf:
                                    exact sequential order), blas2.py:113-162; the
                                    reference's default MultiGrid smoother */

#define MRS_SGS_SYMMETRIC 0      /* forward then backward half-sweep */
#define MRS_SGS_FORWARD   1
#define MRS_SGS_BACKWARD  2

typedef struct {
    int32_t kind;        /* MRS_SMOOTH_* */
    int32_t sweeps;      /* Jacobi: sweeps per application (max_iters) */
    double  weight;      /* Jacobi omega */
    int32_t order;       /* Chebyshev polynomial order */
    int32_t direction;   /* Gauss-Seidel: MRS_SGS_* */
} mrs_smoother;

typedef struct {
    int32_t method;      /* MRS_METHOD_* */
    int32_t precond;     /* MRS_PC_* */
    int64_t nrows;       /* fine rows */
    int64_t m;           /* right-hand sides */
    double  rel_tol;
    int32_t max_iters;
    double  pc_weight;   /* Jacobi preconditioner omega */
    int32_t pc_sweeps;   /* Jacobi preconditioner sweeps */
    int32_t mg_cycles;   /* V-cycles per preconditioner application */
    mrs_smoother pre, post;
    int32_t nlevels;     /* MultiGrid: hierarchy depth (>= 1) */
    int32_t exec;        /* 0: CUDA graph with device-side while loop (default)
                            1: eager launches, host checks convergence
                            2: one captured body graph per iteration, host
                               checks convergence (automatic fallback of 0) */
    int32_t merged;      /* BiCGStab merged=1 (solvers.py:258-283): ||s|| always
                            replaces rnorm in the omega breakdown test */
    double  drift_limit; /* PBiCGStab: ||true r|| / ||recurrence r|| above this raises
                            MRS_ERR_INSTABILITY (solvers.py:68, :415-423); 0 = 1e3 */
    int32_t pc_direction;/* MRS_PC_SGS: MRS_SGS_* (sweeps = pc_sweeps) */
    int32_t vec32;       /* MultiGrid, single GPU: 1 = the V-cycle vectors of levels
                            1 .. (collapsed tail or coarsest) - 1 are float32 (loads
                            widened, fp64 accumulation, stores rounded); the Krylov
                            vectors and level 0 stay float64.  2 = level 0 of the
                            V-cycle too: the whole preconditioner runs on float32
                            vectors (r is rounded on entry, z widened on exit), only
                            the Krylov vectors stay float64 */
} mrs_plan_desc;

typedef struct mrs_plan mrs_plan;

int  mrs_plan_create(const mrs_plan_desc* desc, mrs_plan** out);
/* Upload level `l` (copied; host arrays may be freed afterwards).  For the
 * Jacobi / no-preconditioner plans only level 0 (A) is set.  P, R NULL on the
 * coarsest level.  lmin/lmax: Chebyshev bounds (ignored for Jacobi). */
int  mrs_plan_set_level(mrs_plan* p, int32_t l, const mrs_host_csr* A,
                        const mrs_host_csr* P, const mrs_host_csr* R,
                        double lmin, double lmax);
/* Coarsest-level dense inverse, row-major nc x nc float64 (host). */
int  mrs_plan_set_coarse_inverse(mrs_plan* p, const double* inv, int64_t nc);
/* Collapsed V-cycle tail (MultiGrid plans, single GPU): level `l` (1 <= l <
 * nlevels-1) and everything below it, entered with a zero guess, is the
 * dense row-major n x n float64 operator `op` (n = rows of level l; built at
 * setup by applying the sub-V-cycle to the unit vectors, amg.py
 * vcycle_tail_operator).  The solve then runs x_l = op b_l as ONE launch in
 * place of the level's smoother / residual / transfer kernels and those of
 * every coarser level (replaces solvers.py:651-664 below level l). */
int  mrs_plan_set_dense_tail(mrs_plan* p, int32_t l, const double* op, int64_t n);
int  mrs_plan_finalize(mrs_plan* p, void* stream);

typedef struct {
    int32_t iterations;
    int32_t status;          /* MRS_OK, MRS_ERR_BREAKDOWN or MRS_ERR_INSTABILITY */
    int32_t breakdown_column;
    int32_t breakdown_site;  /* which coefficient vanished (see solver.cu) */
    double  device_ms;       /* device time of the solve (CUDA events) */
} mrs_stats;

/* Solve A X = B.  B, X: (nrows, m) float64, device pointers unless
 * host_buffers != 0 (then pinned/pageable host memory, copies inside).
 * x_is_zero: X is a certified zero initial guess (reference VectorFlags.zero).
 * final_rel (m), history ((max_iters+1) * m, may be NULL) are host outputs. */
int  mrs_plan_solve(mrs_plan* p, const double* B, double* X, int32_t x_is_zero,
                    int32_t host_buffers, void* stream, mrs_stats* stats,
                    double* final_rel, double* history);
/* Algorithmic HBM bytes of one outer iteration / of the setup residual
 * (the roofline model of SURVEY.md 8(d)). */
/* ---- multi-GPU: one process per GPU, NCCL over NVLink --
 * Every level is row-partitioned (local CSR blocks with columns renumbered
 * [own rows | halo rows by (owner, global id)], so each row keeps its global
 * entry order) until it is small enough to be agglomerated: its restriction
 * is computed slice-wise and all-gathered, and the rest of the V-cycle runs
 * replicated.  Dots: local partials -> ncclAllReduce -> device epilogue. */
typedef struct mrs_comm mrs_comm;
int  mrs_comm_unique_id(void* out128);                 /* ncclGetUniqueId */
int  mrs_comm_create(const void* id128, int32_t rank, int32_t nranks, mrs_comm** out);
void mrs_comm_destroy(mrs_comm* c);
/* TEST-ONLY: nranks communicators of ONE process on ONE device joined by an
 * in-process loopback transport (host barriers, stream events, D2D copies)
 * instead of NCCL; out[r] = rank r's.  Each rank's plan is driven by its own
 * host thread and stream in eager exec mode.  Lets the N-rank device path
 * (pack kernel, halo offsets, split reductions, agglomeration all-gathers)
 * run on one GPU; the product's GpuTeam never creates one. */
int  mrs_comm_create_loopback(int32_t nranks, mrs_comm** out);
int  mrs_plan_set_comm(mrs_plan* p, mrs_comm* c);      /* before set_halo / finalize */
/* Level layout: replicated (agglomerated) levels hold every row; the first
 * replicated level after a partitioned one receives its restricted vector as
 * equal slices [slice_row0, slice_row0 + slice_rows) all-gathered. */
int  mrs_plan_set_layout(mrs_plan* p, int32_t l, int32_t replicated, int64_t slice_row0,
                         int64_t slice_rows);
/* Halo of the gathered operand of A_l (which 0), R_l (1) or P_l (2): the
 * local rows to send, grouped by destination rank (counts per rank), and the
 * rows received from each rank (they land after the operand's own rows). */
int  mrs_plan_set_halo(mrs_plan* p, int32_t l, int32_t which, int64_t nsend,
                       const int32_t* send_idx, const int32_t* send_counts,
                       const int32_t* recv_counts);

/* Interior rows [ilo, ihi) of the consumer block of halo `which` (0 A_l,
 * 1 R_l, 2 P_l): rows that read no halo column.  Their product runs while
 * the exchange is in flight (knob "halo_overlap"); the rest after it. */
int  mrs_plan_set_interior(mrs_plan* p, int32_t l, int32_t which, int64_t ilo, int64_t ihi);

double mrs_plan_iteration_bytes(const mrs_plan* p);
/* Warm per-launch device times (us) of one iteration body, each launch
 * bracketed by CUDA events (diagnostics; call after one mrs_plan_solve). */
/* B: right-hand sides (device, nrows x m) to profile with, or NULL = the plan's
 * staging buffer (the last host / staged solve's B). */
int  mrs_plan_profile(mrs_plan* p, const double* B, int32_t iters, void* stream, double* us,
                      int32_t cap,
                      int32_t* count);
/* Diagnostics: kernel name (mangled) of iteration-body launch `idx` (the
 * order of mrs_plan_profile). */
int  mrs_plan_launch_name(mrs_plan* p, int32_t idx, char* buf, int32_t len);
int  mrs_plan_kernel_count(const mrs_plan* p);   /* kernels per outer iteration */
int  mrs_plan_fixed_kernel_count(const mrs_plan* p); /* kernels outside the loop */
void mrs_plan_destroy(mrs_plan* p);

/* ---- 3. native host setup (src/amg.py:55-308, src/solvers.py:486-517) --- */

typedef struct {
    double  strength_threshold;   /* 0.25 */
    int32_t agg_num_levels;       /* 0 */
    int32_t num_paths;            /* 1 */
    int64_t coarse_matrix_size;   /* 500 */
    int32_t max_levels;           /* 25 */
    double  stall_ratio;          /* 0.9 */
    int32_t mixed_precision;      /* levels >= 1 stored float32 */
} mrs_amg_params;

typedef struct mrs_hierarchy mrs_hierarchy;

int  mrs_amg_setup(const mrs_host_csr* A, const mrs_amg_params* prm, mrs_hierarchy** out);
int  mrs_hier_nlevels(const mrs_hierarchy* h);
/* which: 0 = A, 1 = P, 2 = R.  Returns MRS_ERR_ARG when absent.  Arrays stay
 * owned by the hierarchy (int64 row_ptr, uint32 columns before width
 * compression is applied by the caller, float64/float32 values). */
int  mrs_hier_get(const mrs_hierarchy* h, int32_t level, int32_t which, mrs_host_csr* out);
void mrs_hier_destroy(mrs_hierarchy* h);

/* Power-iteration bounds of D^-1 A exactly as solvers.estimate_eig_bounds. */
int  mrs_eig_bounds(const mrs_host_csr* A, int32_t iterations, uint64_t seed_unused,
                    const double* start_vec, double* lmin, double* lmax);

const char* mrs_status_string(int32_t status);
int  mrs_version(void);
/* Tuning knobs, read when a plan captures its graph:
 *   "pdl"       0/1   programmatic dependent launch of the solve-path kernels
 *   "halo_overlap" 0/1/2  multi-GPU: interior rows of a product run while its
 *                   halo exchange is in flight (default 1; 2 = test mode: every
 *                   product with an interior range, halo or not, any size)
 *   "spmm_long_rows" N  operators with <= N rows and >= 12 entries per row run the
 *                   SpMM with 16 entries in flight per lane (default 20000; 0: off)
 *   "coarse_rows" N  rows per CTA of the dense coarse solve (default 1)
 *   "spmm_chunk_rows" N  rows per CTA chunk of the SpMM grid (default 64)
 *   "spmm_long_split" 0/1  rows far longer than their operator's mean run on
 *                   whole CTAs (default 1; solver levels only)
 *   "spmm_coop" 0/1/2  load a row's entries once per lane group and shuffle them:
 *                   1 = operators with >= 12 entries per row (outside the LONG range),
 *                   2 = (default) only long uniform rows (>= 20 per row, max <= 1.1 x mean;
 *                   27-point stencils), 0 = off
 *   "spmm_variant" 0..5  force one SpMM variant for every operator (A/B runs):
 *                   0 = per operator (default), 1 = lane, 2 = cooperative loads,
 *                   3 = 16 entries in flight, 4 = gathers through L2 only,
 *                   5 = gathers with L1::no_allocate
 *   "spmm_autotune" 0/1  plugin calls: measure the variants of an operator on its
 *                   first call per m (default 1; env MRS_SPMM_AUTOTUNE)
 *   "plan_autotune" 0/1  solver plans: the same measurement for every level
 *                   operator at finalize (default 0: the shape heuristic)
 * (Measured-and-rejected variants are listed in profiles/r01_ab_experiments.txt.) */
/* (round 2 keys: "spmm_pair" 0/1/2 pair loads on long-row operators, default 2;
 *  "spmm_variant" 0..7 force one SpMM variant (6 = m=1 stream kernel, 7 = pair loads);
 *  "setup_gpu" 0/1 Galerkin products of mrs_amg_setup on the GPU, default 1) */
int  mrs_set_option(const char* key, int64_t value);

#ifdef __cplusplus
}
#endif
#endif /* MRSOLVE_B200_H */
