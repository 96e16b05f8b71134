// capi.cu -- the kernel-plugin half of the C ABI (include/mrsolve_b200.h).
//
// Each entry point replaces one function of the reference plugin module
// `mrsolve.kernels` (src/kernels/__init__.py:27-41).  Argument checks that
// the reference performs in blas/blas2 (shape, alias, mode) are done here
// because this is the library boundary; everything else is asynchronous on
// the caller's stream.
#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <utility>
#include <vector>

#include "dispatch.h"
#include "sgs.cuh"
#include "sgs_sched.h"
#include "spgemm.h"

using namespace mrs;

namespace {

// 16-byte alignment needed by the vectorised column slices.
inline bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

inline bool m_ok(int64_t m) { return m >= 1 && m <= kMaxM; }

struct Scratch {
    double* partials = nullptr;
    unsigned int* ticket = nullptr;
    int cap = 0;
};

// One reduction scratch (CTA partials + last-CTA ticket) per (device,
// stream): calls on one stream are ordered, so they can share it; calls on
// different streams may run concurrently and must not (the ticket protocol of
// finish_reduction assumes one reduction at a time per scratch).
std::mutex g_scratch_mu;
std::map<std::pair<int, uintptr_t>, Scratch> g_scratch;

int get_scratch(int64_t Km, void* stream, Scratch** out) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return MRS_ERR_CUDA;
    std::lock_guard<std::mutex> lk(g_scratch_mu);
    Scratch& s = g_scratch[{dev, (uintptr_t)stream}];
    int need = max_grid() * (int)Km;
    if (s.cap < need) {
        if (s.partials) cudaFree(s.partials);     // synchronising: no kernel still uses it
        if (!s.ticket) {
            if (cudaMalloc(&s.ticket, sizeof(unsigned int)) != cudaSuccess) return MRS_ERR_ALLOC;
            if (cudaMemset(s.ticket, 0, sizeof(unsigned int)) != cudaSuccess) return MRS_ERR_CUDA;
        }
        if (cudaMalloc(&s.partials, sizeof(double) * need) != cudaSuccess) return MRS_ERR_ALLOC;
        s.cap = need;
    }
    *out = &s;
    return MRS_OK;
}

// Plugin SpMM calls carry no plan: the variant of an operator is measured on
// its first call with a given m (outside stream capture; the product goes to
// a scratch block, the caller's buffers are untouched) and remembered by the
// operator's device arrays.  A later operator reusing those addresses only
// inherits a speed choice -- every variant computes the same bits.
struct TuneKey {
    const void* rp; const void* ci; const void* v; const void* slab;
    int64_t nrows, nnz, m;
    bool operator<(const TuneKey& o) const {
        return std::tie(rp, ci, v, slab, nrows, nnz, m) <
               std::tie(o.rp, o.ci, o.v, o.slab, o.nrows, o.nnz, o.m);
    }
};
std::mutex g_tune_mu;
std::map<TuneKey, int> g_tuned;

int plugin_variant(const DevCsr& D, const double* x, int64_t m, cudaStream_t s) {
    // (a forced variant -- knob spmm_variant -- is applied by the launcher;
    // nothing is measured or remembered meanwhile)
    if (!spmm_autotune_enabled() || spmm_variant() != SV_AUTO) return SV_AUTO;
    TuneKey k{D.rp, D.ci, D.v, D.slab_base, D.nrows, D.nnz, m};
    {
        std::lock_guard<std::mutex> lk(g_tune_mu);
        auto it = g_tuned.find(k);
        if (it != g_tuned.end()) return it->second;
    }
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone)
        return SV_AUTO;
    double* scratch = nullptr;
    if (cudaMalloc(&scratch, sizeof(double) * (size_t)D.nrows * m) != cudaSuccess) {
        cudaGetLastError();
        return SV_AUTO;
    }
    const int64_t fn = (160ll << 20) / 8;           // cold-cache tuning (see spmm_tune)
    double* flush = nullptr;
    if (cudaMalloc(&flush, fn * 8) != cudaSuccess) { cudaGetLastError(); flush = nullptr; }
    else cudaMemsetAsync(flush, 0, fn * 8, s);
    const int v = spmm_tune(D, x, scratch, m, s, nullptr, VP_DD, flush, flush ? fn : 0, 0.97f);
    cudaStreamSynchronize(s);
    cudaFree(scratch);
    if (flush) cudaFree(flush);
    std::lock_guard<std::mutex> lk(g_tune_mu);
    g_tuned[k] = v;
    return v;
}

int vec_call(int op, VArgs a, int K, double* out, void* stream) {
    if (a.n < 0 || !m_ok(a.m)) return MRS_ERR_ARG;
    if (a.n == 0) {
        if (K && out) {
            if (cudaMemsetAsync(out, 0, sizeof(double) * K * a.m, (cudaStream_t)stream) != cudaSuccess)
                return MRS_ERR_CUDA;
        }
        return MRS_OK;
    }
    if (K) {
        Scratch* s = nullptr;
        int rc = get_scratch(K * a.m, stream, &s);
        if (rc) return rc;
        a.red.partials = s->partials;
        a.red.ticket = s->ticket;
        a.red.out = out;
        a.red.st = nullptr;
        a.red.epi = EPI_NONE;
    }
    return launch_vec(op, a, (cudaStream_t)stream) == cudaSuccess ? MRS_OK : MRS_ERR_CUDA;
}

}  // namespace

extern "C" {

int mrs_version(void) { return 1; }

int64_t mrs_stream_launches(void) { return spmm_stream_launches(); }
int64_t mrs_galerkin_gpu_count(void) { return galerkin_gpu_count(); }

// Tuning knobs.  "pdl": launch the solve-path kernels with programmatic
// dependent launch (default 0; env MRS_PDL=1).  Plans capture their graph at
// the first solve, so set options before preparing.
int mrs_set_option(const char* key, int64_t value) {
    if (!key) return MRS_ERR_ARG;
    if (!strcmp(key, "pdl")) { set_pdl((int)value); return MRS_OK; }
    if (!strcmp(key, "coarse_rows")) { set_coarse_rows(value); return MRS_OK; }
    if (!strcmp(key, "spmm_long_rows")) { set_spmm_long_rows(value); return MRS_OK; }
    if (!strcmp(key, "spmm_chunk_rows")) { set_spmm_chunk_rows(value); return MRS_OK; }
    if (!strcmp(key, "spmm_long_split")) { set_spmm_long_split(value); return MRS_OK; }
    if (!strcmp(key, "plan_autotune")) { set_plan_autotune(value); return MRS_OK; }
    if (!strcmp(key, "spmm_autotune")) { set_spmm_autotune(value); return MRS_OK; }
    if (!strcmp(key, "spmm_variant")) { set_spmm_variant(value); return MRS_OK; }
    if (!strcmp(key, "halo_overlap")) { set_halo_overlap(value); return MRS_OK; }
    if (!strcmp(key, "spmm_coop")) { set_spmm_coop(value); return MRS_OK; }
    if (!strcmp(key, "spmm_pair")) { set_spmm_pair(value); return MRS_OK; }
    if (!strcmp(key, "dense_mma")) { set_dense_mma(value); return MRS_OK; }
    if (!strcmp(key, "loop_unroll")) { set_loop_unroll(value); return MRS_OK; }
    if (!strcmp(key, "setup_gpu")) { set_setup_gpu(value); return MRS_OK; }
    return MRS_ERR_ARG;
}

const char* mrs_status_string(int32_t s) {
    switch (s) {
    case MRS_OK: return "ok";
    case MRS_ERR_ARG: return "invalid argument (shape, dtype, mode or alias)";
    case MRS_ERR_CUDA: return "CUDA runtime error";
    case MRS_ERR_UNSUPPORTED: return "configuration not supported on the device path";
    case MRS_ERR_ALLOC: return "allocation failed";
    case MRS_ERR_BREAKDOWN: return "Krylov breakdown";
    case MRS_ERR_SINGULAR: return "zero or missing diagonal entry";
    case MRS_ERR_DEGENERATE: return "AMG setup degeneracy";
    case MRS_ERR_STATE: return "call out of order";
    case MRS_ERR_INSTABILITY: return "pipelined BiCGStab residual recurrence drifted from the true residual";
    }
    return "unknown status";
}

static int spmv_common(const mrs_csr* A, const double* x, double* y, int64_t m, int32_t mode,
                       const double* b, void* stream, int vp);

// _ckernels.pyx:30-57
int mrs_csr_spmv(const mrs_csr* A, const double* x, double* y, int64_t m, int32_t mode,
                 const double* b, void* stream) {
    return spmv_common(A, x, y, m, mode, b, stream, VP_DD);
}

// The same product on float32 block vectors (an extension: the reference's vectors
// are always float64): loads widened, accumulation in float64 in CSR entry order,
// ONE rounding at the store -- y = float(acc).  m in {1, 2, 4, 8, 16, 32}.
int mrs_csr_spmv_f32(const mrs_csr* A, const float* x, float* y, int64_t m, int32_t mode,
                     const float* b, void* stream) {
    if (m < 1 || m > 32 || (m & (m - 1)) != 0) return MRS_ERR_UNSUPPORTED;
    if (A && A->idx_bytes == 1) return MRS_ERR_UNSUPPORTED;
    if (!aligned16(x) || !aligned16(y) || (b && !aligned16(b))) return MRS_ERR_UNSUPPORTED;
    return spmv_common(A, reinterpret_cast<const double*>(x), reinterpret_cast<double*>(y), m, mode,
                       reinterpret_cast<const double*>(b), stream, VP_FF);
}

static int spmv_common(const mrs_csr* A, const double* x, double* y, int64_t m, int32_t mode,
                       const double* b, void* stream, int vp) {
    if (!A || !m_ok(m) || mode < 0 || mode > 3) return MRS_ERR_ARG;
    if (A->idx_bytes != 1 && A->idx_bytes != 2 && A->idx_bytes != 4) return MRS_ERR_ARG;
    if (A->val_bytes != 4 && A->val_bytes != 8) return MRS_ERR_ARG;
    if (A->nrows < 0 || A->nnz < 0 || A->nnz > INT32_MAX) return MRS_ERR_ARG;
    if (mode == MRS_MODE_RSUB && !b) return MRS_ERR_ARG;
    if (x == y) return MRS_ERR_ARG;          // spmv output must not alias the input
    if (A->nrows == 0) return MRS_OK;
    DevCsr D;
    D.nrows = A->nrows; D.ncols = A->ncols; D.nnz = A->nnz;
    D.rp = const_cast<int32_t*>(A->row_ptr);
    D.ci = const_cast<void*>(A->col_idx);
    D.v = const_cast<void*>(A->values);
    D.ib = A->idx_bytes; D.vb = A->val_bytes;
    if (A->slab_base) {
        if (A->idx_bytes != 2 || A->slab_shift < 0 || A->slab_shift > 30) return MRS_ERR_ARG;
        D.slab_base = const_cast<int32_t*>(A->slab_base);
        D.slab_shift = A->slab_shift;
    }
    if (A->long_rows && A->n_long > 0) {
        if (A->long_thr < 1) return MRS_ERR_ARG;
        D.long_rows = const_cast<int32_t*>(A->long_rows);
        D.n_long = A->n_long;
        D.long_thr = A->long_thr;
    }
    D.band = A->band;
    D.blk_max = A->blk_max;
    D.padded = (A->flags & 1) != 0;
    // unaligned views fall back to the scalar-per-column kernel
    bool vec_ok = aligned16(x) && aligned16(y) && (!b || aligned16(b));
    if (vec_ok && vp == VP_DD) D.variant = plugin_variant(D, x, m, (cudaStream_t)stream);
    SpArgs a;
    memset(&a, 0, sizeof(a));
    a.x = x; a.y = y; a.b = b; a.mode = mode; a.vp = vp;
    cudaError_t e = launch_spmm(OP_SPMV, D, a, m, (cudaStream_t)stream, !vec_ok && m > 1);
    return e == cudaSuccess ? MRS_OK : MRS_ERR_CUDA;
}

// _ckernels.pyx:60-79 (gs_sweep): one Gauss-Seidel half-sweep over all rows in
// the sequential order, v = b - c, v -= a_ik x_k (k != diag_pos), x_i = v / a_ii.
// Synchronous on `stream`: the level schedule (sgs_sched.h) is built on the
// host from the device structure on every call; solver plans build theirs once.
int mrs_gs_sweep(const mrs_csr* A, const int64_t* diag_pos, const double* b, const double* c,
                 double* x, int64_t m, int32_t forward, void* stream) {
    if (!A || !diag_pos || !b || !c || !x || m < 1 || m > kThreads) return MRS_ERR_ARG;
    if (A->idx_bytes != 1 && A->idx_bytes != 2 && A->idx_bytes != 4) return MRS_ERR_ARG;
    if (A->val_bytes != 4 && A->val_bytes != 8) return MRS_ERR_ARG;
    if (A->nrows < 0 || A->nnz < 0 || A->nnz > INT32_MAX || A->ncols != A->nrows) return MRS_ERR_ARG;
    if (A->slab_base && (A->idx_bytes != 2 || A->slab_shift < 0 || A->slab_shift > 30))
        return MRS_ERR_ARG;
    if (m % 2 == 0 && !(aligned16(b) && aligned16(c) && aligned16(x))) return MRS_ERR_ARG;
    const int64_t n = A->nrows, nnz = A->nnz;
    if (n == 0) return MRS_OK;
    cudaStream_t s = (cudaStream_t)stream;
    MRS_CUDA_OK(cudaStreamSynchronize(s));
    std::vector<int32_t> rp32(n + 1);
    std::vector<uint8_t> ci((size_t)nnz * A->idx_bytes), vals((size_t)nnz * A->val_bytes);
    std::vector<int64_t> dp(n);
    std::vector<int32_t> sb;
    MRS_CUDA_OK(cudaMemcpy(rp32.data(), A->row_ptr, (n + 1) * 4, cudaMemcpyDeviceToHost));
    MRS_CUDA_OK(cudaMemcpy(ci.data(), A->col_idx, ci.size(), cudaMemcpyDeviceToHost));
    MRS_CUDA_OK(cudaMemcpy(vals.data(), A->values, vals.size(), cudaMemcpyDeviceToHost));
    MRS_CUDA_OK(cudaMemcpy(dp.data(), diag_pos, n * 8, cudaMemcpyDeviceToHost));
    if (A->slab_base) {
        sb.resize(((n - 1) >> A->slab_shift) + 1);
        MRS_CUDA_OK(cudaMemcpy(sb.data(), A->slab_base, sb.size() * 4, cudaMemcpyDeviceToHost));
    }
    std::vector<int64_t> rp(rp32.begin(), rp32.end());
    const int ib = A->idx_bytes;
    auto col = [&](int64_t i, int64_t k) -> int64_t {
        int64_t cc = ib == 4 ? ((const uint32_t*)ci.data())[k]
                   : ib == 2 ? ((const uint16_t*)ci.data())[k] : ci[k];
        return A->slab_base ? cc + sb[i >> A->slab_shift] : cc;
    };
    std::vector<int32_t> dp32(n), order, lptr, ci16;
    std::vector<double> d(n);
    for (int64_t i = 0; i < n; ++i) {
        if (dp[i] < rp[i] || dp[i] >= rp[i + 1]) return MRS_ERR_ARG;
        dp32[i] = (int32_t)dp[i];
        d[i] = A->val_bytes == 8 ? ((const double*)vals.data())[dp[i]]
                                 : (double)((const float*)vals.data())[dp[i]];
    }
    sgs_levels(n, rp.data(), col, forward ? 0 : 1, order, lptr);
    std::vector<int4> meta(n);
    for (int64_t q = 0; q < n; ++q) {
        const int32_t i = order[q];
        meta[q] = make_int4(i, rp32[i], rp32[i + 1], dp32[i]);
    }
    // temporaries: schedule, diagonal, u8 columns widened to u16
    void* buf[4] = {nullptr, nullptr, nullptr, nullptr};
    auto release = [&]() { for (void* q : buf) if (q) cudaFree(q); };
    const size_t sz[4] = {meta.size() * sizeof(int4), lptr.size() * 4, (size_t)n * 8,
                          ib == 1 ? (size_t)nnz * 2 : 0};
    for (int q = 0; q < 4; ++q)
        if (sz[q] && cudaMalloc(&buf[q], sz[q]) != cudaSuccess) { release(); return MRS_ERR_ALLOC; }
    const void* cols = A->col_idx;
    int ibd = ib;
    bool ok = cudaMemcpy(buf[0], meta.data(), sz[0], cudaMemcpyHostToDevice) == cudaSuccess &&
              cudaMemcpy(buf[1], lptr.data(), sz[1], cudaMemcpyHostToDevice) == cudaSuccess &&
              cudaMemcpy(buf[2], d.data(), sz[2], cudaMemcpyHostToDevice) == cudaSuccess;
    if (ok && ib == 1) {
        std::vector<uint16_t> w(ci.begin(), ci.end());
        ok = cudaMemcpy(buf[3], w.data(), sz[3], cudaMemcpyHostToDevice) == cudaSuccess;
        cols = buf[3];
        ibd = 2;
    }
    if (!ok) { release(); return MRS_ERR_CUDA; }
    SgsArgs a;
    memset(&a, 0, sizeof(a));
    a.rp = A->row_ptr; a.ci = cols; a.vals = A->values;
    a.slab_base = A->slab_base; a.slab_shift = A->slab_shift;
    a.meta = (const int4*)buf[0]; a.lptr = (const int32_t*)buf[1];
    a.nlev = (int)lptr.size() - 1;
    a.d = (const double*)buf[2];
    a.b = b; a.c = c; a.x = x; a.m = (int)m; a.nrows = (int)n;
    cudaError_t e = launch_sgs(a, A->val_bytes, ibd, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    release();
    return e == cudaSuccess ? MRS_OK : MRS_ERR_CUDA;
}

int mrs_axpby(int64_t n, int64_t m, const double* a, const double* x, const double* b,
              double* y, void* stream) {
    VArgs A; memset(&A, 0, sizeof(A));
    A.n = n; A.m = m; A.a = a; A.b = b; A.x = x; A.y = y;
    return vec_call(V_AXPBY, A, 0, nullptr, stream);
}

int mrs_add2_scaled(int64_t n, int64_t m, double* y, const double* a, const double* u,
                    const double* b, const double* v, void* stream) {
    VArgs A; memset(&A, 0, sizeof(A));
    A.n = n; A.m = m; A.y = y; A.a = a; A.u = u; A.b = b; A.v = v;
    return vec_call(V_ADD2, A, 0, nullptr, stream);
}

int mrs_fused_paired_update(int64_t n, int64_t m, double* y1, const double* a,
                            const double* u, const double* b, const double* s, double* y2,
                            const double* c, const double* w, void* stream) {
    if (y2 == s || y2 == w || y1 == y2) return MRS_ERR_ARG;
    VArgs A; memset(&A, 0, sizeof(A));
    A.n = n; A.m = m; A.y = y1; A.a = a; A.u = u; A.b = b; A.s = s; A.y2 = y2; A.c = c; A.w = w;
    return vec_call(V_PAIRED, A, 0, nullptr, stream);
}

int mrs_dot(int64_t n, int64_t m, const double* x, const double* y, double* out, void* stream) {
    VArgs A; memset(&A, 0, sizeof(A));
    A.n = n; A.m = m; A.x = x; A.z = y;
    return vec_call(V_DOT, A, 1, out, stream);
}

int mrs_fused_update_dot(int64_t n, int64_t m, const double* a, const double* x,
                         const double* b, double* y, double* out, void* stream) {
    VArgs A; memset(&A, 0, sizeof(A));
    A.n = n; A.m = m; A.a = a; A.x = x; A.b = b; A.y = y;
    return vec_call(V_UPDATE_DOT, A, 1, out, stream);
}

int mrs_fused_update_dot2(int64_t n, int64_t m, double* y, const double* u, const double* c,
                          const double* w, const double* z, double* d1, double* d2,
                          void* stream) {
    if (!d1 || !d2) return MRS_ERR_ARG;
    VArgs A; memset(&A, 0, sizeof(A));
    A.n = n; A.m = m; A.y = y; A.u = u; A.c = c; A.w = w; A.z = z;
    // results land as [d1 | d2] in scratch, then split
    double* tmp = nullptr;
    int rc;
    if (cudaMallocAsync(&tmp, sizeof(double) * 2 * m, (cudaStream_t)stream) != cudaSuccess)
        return MRS_ERR_ALLOC;
    rc = vec_call(V_UPDATE_DOT2, A, 2, tmp, stream);
    if (rc == MRS_OK) {
        cudaStream_t s = (cudaStream_t)stream;
        if (cudaMemcpyAsync(d1, tmp, sizeof(double) * m, cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
            cudaMemcpyAsync(d2, tmp + m, sizeof(double) * m, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
            rc = MRS_ERR_CUDA;
    }
    cudaFreeAsync(tmp, (cudaStream_t)stream);
    return rc;
}

}  // extern "C"
