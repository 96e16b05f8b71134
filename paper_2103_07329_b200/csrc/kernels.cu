// kernels.cu -- template instantiation and dispatch of the SpMM and vector
// kernel families, and the dense coarse-level solve.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <mutex>
#include <unordered_map>

#include "launch.cuh"

namespace mrs {

int max_grid() { return num_sms() * kMaxGridPerSM; }

// Tuning knobs (mrs_set_option): read at launch / capture time.
static int g_pdl = -1;


bool pdl_enabled() {
    if (g_pdl < 0) {
        const char* e = getenv("MRS_PDL");
        g_pdl = (e && e[0] == '1') ? 1 : 0;
    }
    return g_pdl == 1;
}

void set_pdl(int on) { g_pdl = on ? 1 : 0; }

static int64_t g_long_rows = 20000;   // A/B: profiles/r01_ab_experiments.txt
int64_t spmm_long_max_rows() { return g_long_rows; }
void set_spmm_long_rows(int64_t v) { g_long_rows = v < 0 ? 0 : v; }
static int64_t g_chunk_rows = 64;     // A/B: profiles/r01_ab_experiments.txt
int64_t spmm_chunk_rows() { return g_chunk_rows; }
void set_spmm_chunk_rows(int64_t v) { g_chunk_rows = v < 1 ? 1 : v; }
static int64_t g_long_split = 1;      // long rows by whole CTAs (0: lane path only)
int64_t spmm_long_split() { return g_long_split; }
void set_spmm_long_split(int64_t v) { g_long_split = v ? 1 : 0; }
static int64_t g_loop_unroll = 4;     // CG bodies of <= 4 kernels: iterations per WHILE trip
int64_t loop_unroll() { return g_loop_unroll; }
void set_loop_unroll(int64_t v) { g_loop_unroll = v < 1 ? 1 : (v > 8 ? 8 : v); }
static int64_t g_dense_mma = 1;       // FP64 tensor-core dense tail (dense_mma_kernel)
bool dense_mma_enabled() { return g_dense_mma != 0; }
void set_dense_mma(int64_t v) { g_dense_mma = v ? 1 : 0; }
static int64_t g_halo_overlap = 1;    // multi-GPU: interior rows during the exchange
int64_t halo_overlap() { return g_halo_overlap; }
void set_halo_overlap(int64_t v) { g_halo_overlap = v < 0 ? 0 : (v > 2 ? 2 : v); }
static int64_t g_variant = 0;         // 0: per operator (autotuned / heuristic)
int64_t spmm_variant() { return g_variant; }
void set_spmm_variant(int64_t v) { g_variant = v < 0 ? 0 : (v > 7 ? 0 : v); }
// pair loads for operators with >= 12 entries per row (knob spmm_pair, env MRS_SPMM_PAIR):
// 0 off, 1 instead of the plain lane kernel, 2 also instead of the cooperative one
static int64_t g_pair = -1;
int64_t spmm_pair() {
    if (g_pair < 0) {
        const char* e = getenv("MRS_SPMM_PAIR");
        g_pair = e ? atoi(e) : 2;
        if (g_pair < 0 || g_pair > 2) g_pair = 2;
    }
    return g_pair;
}
void set_spmm_pair(int64_t v) { g_pair = v < 0 ? 0 : (v > 2 ? 2 : v); }
static int64_t g_coop = 2;            // cooperative entry loads (A/B: profiles/r01_ab_experiments.txt)
int64_t spmm_coop() { return g_coop; }
void set_spmm_coop(int64_t v) { g_coop = v < 0 ? 0 : (v > 2 ? 2 : v); }

int spmm_grid(int64_t nrows, int64_t m) {   // upper bound (scratch sizing)
    (void)nrows; (void)m;
    return max_grid();
}

int vec_grid(int64_t n, int64_t m) {
    (void)n; (void)m;
    return max_grid();
}

cudaError_t launch_spmm(int op, const DevCsr& A, SpArgs a, int64_t m, cudaStream_t s,
                        bool generic) {
    a.rp = A.rp; a.ci = A.ci; a.vals = A.v; a.m = m; a.nnz_hint = A.nnz;
    a.nrows = a.vrows ? a.vrows : A.nrows;       // split launches: the subset
    a.rows_hint = A.nrows;
    a.ncols_hint = A.ncols;
    a.slab_base = A.slab_base;
    a.slab_shift = A.slab_shift;
    if (!a.xo) a.xo = a.x;
    if (a.row0) {
        // split launch: rows [row0, row0 + vrows) through offset row-indexed
        // pointers (the kernel itself always starts at row 0); slab bases are
        // per 2^shift rows, so row0 must sit on a slab boundary
        const int64_t r0 = a.row0;
        if (A.n_long || (A.slab_base && (r0 & ((1ll << A.slab_shift) - 1))))
            return cudaErrorInvalidValue;
        const size_t eo = (size_t)r0 * m;            // element offset of row r0
        const bool y32 = a.vp == VP_FF || a.vp == VP_DF;
        auto off = [&](auto* p) -> decltype(p) {
            if (!p) return p;
            using T = std::remove_cv_t<std::remove_pointer_t<decltype(p)>>;
            (void)sizeof(T);
            return reinterpret_cast<decltype(p)>(reinterpret_cast<std::conditional_t<
                std::is_const_v<std::remove_pointer_t<decltype(p)>>, const char*, char*>>(p) +
                eo * (y32 ? 4 : 8));
        };
        a.rp = A.rp + r0;
        if (A.slab_base) a.slab_base = A.slab_base + (r0 >> A.slab_shift);
        a.y = off(a.y); a.b = off(a.b); a.x_out = off(a.x_out); a.r_out = off(a.r_out);
        a.dv_out = off(a.dv_out); a.x_in = off(a.x_in); a.r_in = off(a.r_in);
        a.seed_out = off(a.seed_out);
        a.xo = off(a.xo);
        if (a.d) a.d = a.d + r0;
    }
    a.max_row_hint = A.max_row;
    a.long_rows = A.long_rows;
    a.n_long = spmm_long_split() ? A.n_long : 0;
    a.long_thr = A.long_thr;
    a.long_ctas = 0;
    if (a.nrows == 0) return cudaSuccess;
    // the SpMM engine indexes with 32 bits (rows, entries, element offsets)
    if ((A.nrows + 1) * m >= (int64_t)INT32_MAX || (A.ncols + 1) * m >= (int64_t)INT32_MAX ||
        A.nnz >= (int64_t)INT32_MAX)
        return cudaErrorInvalidValue;
    a.variant = A.variant;
    if (op == OP_SPMV && (a.variant ? a.variant : (int)spmm_variant()) == SV_STREAM && !generic &&
        spmm_stream_eligible(A, m, a))
        return launch_spmm_stream(A, a, s);
    if (A.vb == 8) {
        switch (op) {
        case OP_SPMV: return launch_spmm_op_f64<OP_SPMV>(A, a, m, s, generic);
        case OP_JAC_SWEEP: return launch_spmm_op_f64<OP_JAC_SWEEP>(A, a, m, s, generic);
        case OP_CHEB_FIRST: return launch_spmm_op_f64<OP_CHEB_FIRST>(A, a, m, s, generic);
        case OP_CHEB_STEP: return launch_spmm_op_f64<OP_CHEB_STEP>(A, a, m, s, generic);
        }
    } else if (A.vb == 4) {
        switch (op) {
        case OP_SPMV: return launch_spmm_op_f32<OP_SPMV>(A, a, m, s, generic);
        case OP_JAC_SWEEP: return launch_spmm_op_f32<OP_JAC_SWEEP>(A, a, m, s, generic);
        case OP_CHEB_FIRST: return launch_spmm_op_f32<OP_CHEB_FIRST>(A, a, m, s, generic);
        case OP_CHEB_STEP: return launch_spmm_op_f32<OP_CHEB_STEP>(A, a, m, s, generic);
        }
    }
    return cudaErrorInvalidValue;
}

// Per-operator SpMM variant choice by measurement: every applicable variant
// (lane / cooperative loads / 16 in flight) runs the operator's product
// y = A x (ASSIGN) back to back on the given buffers and the fastest wins.
// All variants compute the same bits, so the choice only affects speed.
// Returns the SpmmVariant to store in A.variant (SV_AUTO: nothing to choose).
static int64_t g_plan_autotune = 0;
int64_t plan_autotune() { return g_plan_autotune; }
void set_plan_autotune(int64_t v) { g_plan_autotune = v ? 1 : 0; }
static int64_t g_autotune = -1;
int64_t spmm_autotune_enabled() {
    if (g_autotune < 0) {                    // default on; MRS_SPMM_AUTOTUNE=0 for A/B runs
        const char* e = getenv("MRS_SPMM_AUTOTUNE");
        g_autotune = (e && e[0] == '0') ? 0 : 1;
    }
    return g_autotune;
}
void set_spmm_autotune(int64_t v) { g_autotune = v ? 1 : 0; }

// Reads `n` doubles (an L2-sized buffer): evicts the operator's lines so a
// tuning launch sees the cold-cache conditions of a solve, whose V-cycle
// streams far more than the 126 MB L2 between two uses of an operator.
__global__ void l2_flush_kernel(const double* __restrict__ p, int64_t n, double* sink) {
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        acc += __ldcs(p + i);
    if (acc == 1.2345e300) *sink = acc;     // never true: keeps the loads
}

int spmm_tune(const DevCsr& A, const double* x, double* y, int64_t m, cudaStream_t s,
              float* best_us, int vp, const double* flush, int64_t flush_n, float keep) {
    if (best_us) *best_us = 0.f;
    if (!spmm_autotune_enabled() || A.nrows == 0 || A.nnz == 0 || spmm_variant() != SV_AUTO)
        return SV_AUTO;
    int cand[7], nc = 0;
    cand[nc++] = SV_LANE;
    {
        SpArgs probe;
        memset(&probe, 0, sizeof(probe));
        probe.x = x; probe.y = y; probe.vp = vp;
        if (spmm_stream_eligible(A, m, probe)) cand[nc++] = SV_STREAM;
    }
    if (vp == VP_DD && (m == 4 || m == 8 || m == 16)) cand[nc++] = SV_COOP;
    if (m <= 16 && (m & (m - 1)) == 0) cand[nc++] = SV_LONG;
    if (vp == VP_DD && m <= 16 && (m & (m - 1)) == 0) {
        cand[nc++] = SV_LANE_L2;
        cand[nc++] = SV_LANE_NA;
        if (m >= 2) cand[nc++] = SV_PAIR;
    }
    if (nc == 1) return SV_AUTO;
    constexpr int kReps = 5;
    cudaEvent_t ev[2 * kReps];
    int made = 0;
    for (; made < 2 * kReps; ++made)
        if (cudaEventCreate(&ev[made]) != cudaSuccess) break;
    SpArgs a;
    memset(&a, 0, sizeof(a));
    a.x = x; a.y = y; a.mode = MRS_MODE_ASSIGN; a.vp = vp;
    int best = SV_AUTO;
    float best_t = 3.4e38f;
    float tm[7] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int i = 0; i < nc && made == 2 * kReps; ++i) {
        DevCsr B = A;
        B.variant = cand[i];
        cudaError_t e = launch_spmm(OP_SPMV, B, a, m, s);           // warm-up (instruction cache)
        for (int r = 0; r < kReps && e == cudaSuccess; ++r) {
            if (flush) l2_flush_kernel<<<4 * num_sms(), kThreads, 0, s>>>(flush, flush_n, y);
            cudaEventRecord(ev[2 * r], s);
            e = launch_spmm(OP_SPMV, B, a, m, s);
            cudaEventRecord(ev[2 * r + 1], s);
        }
        if (e != cudaSuccess || cudaEventSynchronize(ev[2 * kReps - 1]) != cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        float t[kReps];
        for (int r = 0; r < kReps; ++r) cudaEventElapsedTime(&t[r], ev[2 * r], ev[2 * r + 1]);
        std::sort(t, t + kReps);
        tm[i] = t[kReps / 2];
        if (t[kReps / 2] < best_t) { best_t = t[kReps / 2]; best = cand[i]; }
    }
    for (int k = 0; k < made; ++k) cudaEventDestroy(ev[k]);
    // The isolated cold launch is only a proxy for the operator's cost inside
    // a solve (other operands, fused epilogues, neighbouring kernels): leave
    // the shape heuristic's choice unless another variant is clearly faster.
    const int dflt = vp == VP_DD ? spmm_shape_variant(A.nrows, A.nnz, A.max_row, m) : SV_LANE;
    for (int i = 0; i < nc; ++i)
        if (cand[i] == dflt && tm[i] > 0.f && best != dflt && best_t > keep * tm[i]) {
            best = dflt;
            best_t = tm[i];
        }
    if (best_us && best != SV_AUTO) *best_us = 1e3f * best_t;
    return best;
}

// fp32 preconditioner interface (plan option vec32 = 2: level 0 of the V-cycle
// stores its vectors in float too): the Krylov residual enters the V-cycle as a
// float right-hand side (+ the level-0 zero-guess smoother seed), the V-cycle's
// float result leaves as the double z.
__global__ void __launch_bounds__(kThreads) cvt_to32_kernel(const double* __restrict__ r,
                                                            float* __restrict__ b32, int64_t n, int m,
                                                            int seed_mode, const double* __restrict__ d,
                                                            double w, float* __restrict__ seed_out,
                                                            const int* guard) {
    pdl_enter();
    if (guard && *guard) return;
    const int64_t total = n * m;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float f = __double2float_rn(r[i]);
        b32[i] = f;
        if (seed_mode) seed_out[i] = __double2float_rn(seed_value(seed_mode, (double)f, __ldg(d + i / m), w));
    }
}
__global__ void __launch_bounds__(kThreads) cvt_from32_kernel(const float* __restrict__ x32,
                                                              double* __restrict__ z, int64_t total,
                                                              const int* guard) {
    pdl_enter();
    if (guard && *guard) return;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x)
        z[i] = (double)x32[i];
}
cudaError_t launch_cvt_to32(const double* r, float* b32, int64_t n, int64_t m, int seed_mode,
                            const double* d, double w, float* seed_out, const int* guard,
                            cudaStream_t s) {
    const int g = (int)std::min<int64_t>((n * m + kThreads - 1) / kThreads, (int64_t)num_sms() * 8);
    (void)launch_ex(cvt_to32_kernel, std::max(g, 1), s, r, b32, n, (int)m, seed_mode, d, w, seed_out,
                    guard);
    return cudaGetLastError();
}
cudaError_t launch_cvt_from32(const float* x32, double* z, int64_t total, const int* guard,
                              cudaStream_t s) {
    const int g = (int)std::min<int64_t>((total + kThreads - 1) / kThreads, (int64_t)num_sms() * 8);
    (void)launch_ex(cvt_from32_kernel, std::max(g, 1), s, x32, z, total, guard);
    return cudaGetLastError();
}

template <int OP>
static cudaError_t vec_op(const VArgs& a, cudaStream_t s) {
    int g;
    int64_t chunk;
    wave_grid((const void*)vec_kernel<OP>, a.n, (int64_t)(kThreads / a.m) * vec_unroll<OP>(), g,
              chunk);
    (void)launch_ex(vec_kernel<OP>, g, s, a, chunk);
    return cudaGetLastError();
}

int vec_op_k(int op) {
    switch (op) {
    case V_DOT: return VK<V_DOT>::K;
    case V_UPDATE_DOT: return VK<V_UPDATE_DOT>::K;
    case V_UPDATE_DOT2: return VK<V_UPDATE_DOT2>::K;
    case V_CG_UPDATE: return VK<V_CG_UPDATE>::K;
    case V_CG_UPDATE_JAC: return VK<V_CG_UPDATE_JAC>::K;
    case V_DOT3: return VK<V_DOT3>::K;
    case V_BICG_XR: return VK<V_BICG_XR>::K;
    case V_DOT2: return VK<V_DOT2>::K;
    case V_DOT5: return VK<V_DOT5>::K;
    case V_PBICG_QY: return VK<V_PBICG_QY>::K;
    case V_PBICG_W: return VK<V_PBICG_W>::K;
    }
    return 0;
}

cudaError_t launch_vec(int op, VArgs a, cudaStream_t s) {
    switch (op) {
    case V_AXPBY: return vec_op<V_AXPBY>(a, s);
    case V_ADD2: return vec_op<V_ADD2>(a, s);
    case V_PAIRED: return vec_op<V_PAIRED>(a, s);
    case V_DOT: return vec_op<V_DOT>(a, s);
    case V_UPDATE_DOT: return vec_op<V_UPDATE_DOT>(a, s);
    case V_UPDATE_DOT2: return vec_op<V_UPDATE_DOT2>(a, s);
    case V_COPY: return vec_op<V_COPY>(a, s);
    case V_CG_UPDATE: return vec_op<V_CG_UPDATE>(a, s);
    case V_CG_UPDATE_JAC: return vec_op<V_CG_UPDATE_JAC>(a, s);
    case V_P_UPDATE: return vec_op<V_P_UPDATE>(a, s);
    case V_SEED: return vec_op<V_SEED>(a, s);
    case V_BICG_P: return vec_op<V_BICG_P>(a, s);
    case V_BICG_S: return vec_op<V_BICG_S>(a, s);
    case V_DOT3: return vec_op<V_DOT3>(a, s);
    case V_BICG_XR: return vec_op<V_BICG_XR>(a, s);
    case V_DOT2: return vec_op<V_DOT2>(a, s);
    case V_DOT5: return vec_op<V_DOT5>(a, s);
    case V_BICG_XR0: return vec_op<V_BICG_XR0>(a, s);
    case V_PBICG_QY: return vec_op<V_PBICG_QY>(a, s);
    case V_PBICG_W: return vec_op<V_PBICG_W>(a, s);
    }
    return cudaErrorInvalidValue;
}

// Coarsest level: x = Ainv b (replaces scipy lu_solve, solvers.py:644-649).
// CTA handles rows_per_cta rows; thread (ks, c) folds k = ks, ks + kpb, ... for
// column c, then the ks partials are folded in order (deterministic).
static int g_coarse_rows = 1;     // rows per CTA of the coarse solve (knob coarse_rows; A/B in profiles)
void set_coarse_rows(int64_t v) { g_coarse_rows = v < 1 ? 1 : (v > 64 ? 64 : (int)v); }

__global__ void __launch_bounds__(kThreads) coarse_kernel(const double* __restrict__ inv, int64_t nc,
                                                          const double* __restrict__ b,
                                                          double* __restrict__ x, int m,
                                                          const int* guard, int rows_per_cta) {
    pdl_enter();
    if (guard && *guard) return;
    __shared__ double s_t[kThreads];
    const int kpb = kThreads / m;
    const int c = threadIdx.x % m, ks = threadIdx.x / m;
    for (int rr = 0; rr < rows_per_cta; ++rr) {
        int64_t i = (int64_t)blockIdx.x * rows_per_cta + rr;
        if (i >= nc) break;
        double acc = 0.0;
        if (ks < kpb)
            for (int64_t k = ks; k < nc; k += kpb)
                acc = add(acc, mul(__ldg(inv + i * nc + k), __ldg(b + k * m + c)));
        s_t[threadIdx.x] = acc;
        __syncthreads();
        if (threadIdx.x < m) {
            double t = s_t[threadIdx.x];
            for (int q = 1; q < kpb; ++q) t = add(t, s_t[q * m + threadIdx.x]);
            x[i * m + threadIdx.x] = t;
        }
        __syncthreads();
    }
}

cudaError_t launch_coarse(const double* inv, int64_t nc, const double* b, double* x,
                          int64_t m, const int* guard, cudaStream_t s) {
    const int rpc = g_coarse_rows;
    int g = (int)((nc + rpc - 1) / rpc);
    (void)launch_ex(coarse_kernel, g, s, inv, nc, b, x, (int)m, guard, rpc);
    return cudaGetLastError();
}

// x = T b for a dense row-major n x n operator T (the collapsed V-cycle
// tail).  A warp owns R consecutive rows and walks k in steps of 32: lane j
// loads T[i_r, k + j] (256 B coalesced per row) and row k + j of b (M
// contiguous doubles) and keeps R x M partial sums; a xor tree over the
// lanes finishes each (row, column).  T is streamed once; b (n*M*8 bytes)
// stays in L1/L2 and is re-read once per R rows.  Fixed reduction shape.
template <int M, int R>
__global__ void __launch_bounds__(kThreads) dense_kernel(const double* __restrict__ T, int64_t n,
                                                         const double* __restrict__ b,
                                                         double* __restrict__ x,
                                                         const int* guard) {
    pdl_enter();
    if (guard && *guard) return;
    const int lane = threadIdx.x % 32;
    const int64_t i0 = ((int64_t)blockIdx.x * (kThreads / 32) + threadIdx.x / 32) * R;
    if (i0 >= n) return;
    const double* Tr[R];
#pragma unroll
    for (int r = 0; r < R; ++r) Tr[r] = T + min(i0 + r, n - 1) * n;
    double acc[R][M];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int c = 0; c < M; ++c) acc[r][c] = 0.0;
    for (int64_t k = lane; k < n; k += 32) {
        double t[R];
#pragma unroll
        for (int r = 0; r < R; ++r) t[r] = __ldg(Tr[r] + k);
        double bv[M];
        if constexpr (M == 1) {
            bv[0] = __ldg(b + k);
        } else {
#pragma unroll
            for (int c = 0; c < M; c += 2) {
                const double2 v = __ldg(reinterpret_cast<const double2*>(b + k * M + c));
                bv[c] = v.x; bv[c + 1] = v.y;
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int c = 0; c < M; ++c) acc[r][c] = add(acc[r][c], mul(t[r], bv[c]));
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int c = 0; c < M; ++c)
                acc[r][c] = add(acc[r][c], __shfl_xor_sync(0xffffffffu, acc[r][c], off));
    if (lane == 0) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (i0 + r >= n) break;
#pragma unroll
            for (int c = 0; c < M; ++c) x[(i0 + r) * M + c] = acc[r][c];
        }
    }
}

cudaError_t launch_coarse(const double* inv, int64_t nc, const double* b, double* x,
                          int64_t m, const int* guard, cudaStream_t s);

// x = T b on the FP64 tensor cores (mma.sync m8n8k4 f64), m = 8 * NT columns.
// A CTA owns 8 rows of T; its 8 warps split k and each accumulates the 8 x 8
// (x NT) output block over its k range with DMMA (A fragment = T[8 rows][4 k],
// B fragment = b[4 k][8 columns]); the 8 partial blocks are folded in warp
// order through shared memory.  T is streamed once; b (n x m) is re-read once
// per 8 rows from L2.  Products are fused multiply-adds (dense tail only: the
// reference-order SpMM kernels never use this).
template <int NT>
__global__ void __launch_bounds__(kThreads) dense_mma_kernel(const double* __restrict__ T, int64_t n,
                                                             const double* __restrict__ b,
                                                             double* __restrict__ x,
                                                             const int* guard) {
    pdl_enter();
    if (guard && *guard) return;
    constexpr int M = 8 * NT;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t4 = lane & 3;
    const int64_t row0 = (int64_t)blockIdx.x * 8;
    const int64_t arow = min(row0 + g, n - 1);
    const double* Ta = T + arow * n;
    // k range of this warp: multiples of 4
    const int64_t nk4 = (n + 3) / 4;
    const int64_t per = (nk4 + 7) / 8;
    const int64_t k0 = (int64_t)warp * per * 4, k1 = min(k0 + per * 4, n);
    double c[NT][2];
#pragma unroll
    for (int j = 0; j < NT; ++j) c[j][0] = c[j][1] = 0.0;
    constexpr int U = 16;  // k-steps in flight (ncu: 4 left the kernel at 26% occupancy, latency-bound)
    for (int64_t k = k0; k < k1; k += 4 * U) {
        double av[U], bv[U][NT];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t kk = k + 4 * u + t4;
            const bool ok = kk < k1;
            av[u] = ok ? __ldg(Ta + kk) : 0.0;
#pragma unroll
            for (int j = 0; j < NT; ++j) bv[u][j] = ok ? __ldg(b + kk * M + 8 * j + g) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int j = 0; j < NT; ++j)
                asm volatile(
                    "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                    : "+d"(c[j][0]), "+d"(c[j][1])
                    : "d"(av[u]), "d"(bv[u][j]));
    }
    __shared__ double s_c[kThreads / 32][8 * M];
#pragma unroll
    for (int j = 0; j < NT; ++j) {
        s_c[warp][g * M + 8 * j + 2 * t4] = c[j][0];
        s_c[warp][g * M + 8 * j + 2 * t4 + 1] = c[j][1];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 8 * M; e += kThreads) {
        const int r = e / M;
        if (row0 + r >= n) continue;
        double acc = s_c[0][e];
        for (int w = 1; w < kThreads / 32; ++w) acc = add(acc, s_c[w][e]);
        x[(row0 + r) * M + (e % M)] = acc;
    }
}

cudaError_t launch_dense(const double* T, int64_t n, const double* b, double* x, int64_t m,
                         const int* guard, cudaStream_t s) {
    constexpr int W = kThreads / 32;
    if (n > 1024 && dense_mma_enabled() && (m == 8 || m == 16)) {
        const int g = (int)((n + 7) / 8);
        if (m == 8) (void)launch_ex(dense_mma_kernel<1>, g, s, T, n, b, x, guard);
        else (void)launch_ex(dense_mma_kernel<2>, g, s, T, n, b, x, guard);
        return cudaGetLastError();
    }
    // small operators: one row per CTA (more CTAs in flight than warp-rows)
    if (n <= 1024) return launch_coarse(T, n, b, x, m, guard, s);
    // rows per warp: the most (<= 32 / M partial sums per lane) that still
    // give every SM a CTA
    auto rows = [&](int rmax) {
        int R = rmax;
        while (R > 1 && (n + (int64_t)R * W - 1) / ((int64_t)R * W) < num_sms()) R >>= 1;
        return R;
    };
    auto go = [&](auto k1, auto k2, auto k4, auto k8, int rmax) {
        const int R = rows(rmax);
        const int64_t warps = (n + R - 1) / R;
        const int g = (int)((warps + W - 1) / W);
        if (R == 8) (void)launch_ex(k8, g, s, T, n, b, x, guard);
        else if (R == 4) (void)launch_ex(k4, g, s, T, n, b, x, guard);
        else if (R == 2) (void)launch_ex(k2, g, s, T, n, b, x, guard);
        else (void)launch_ex(k1, g, s, T, n, b, x, guard);
        return cudaGetLastError();
    };
#define MRS_DK(MM) dense_kernel<MM, 1>, dense_kernel<MM, 2>, dense_kernel<MM, (MM <= 8 ? 4 : 2)>, \
                   dense_kernel<MM, (MM <= 4 ? 8 : 2)>
    switch (m) {
    case 1: return go(MRS_DK(1), 8);
    case 2: return go(MRS_DK(2), 8);
    case 4: return go(MRS_DK(4), 8);
    case 8: return go(MRS_DK(8), 4);
    case 16: return go(MRS_DK(16), 2);
    default: return launch_coarse(T, n, b, x, m, guard, s);   // any m
    }
#undef MRS_DK
}

}  // namespace mrs
