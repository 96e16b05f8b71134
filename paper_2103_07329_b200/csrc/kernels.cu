// kernels.cu -- template instantiation and dispatch of the SpMM and vector
// kernel families, and the dense coarse-level solve.
#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "dispatch.h"

namespace mrs {

int max_grid() { return num_sms() * kMaxGridPerSM; }

// Tuning knobs (mrs_set_option): read at launch / capture time.
static int g_pdl = -1;
static int g_staged = 1;

void set_staged(int on) { g_staged = on ? 1 : 0; }

bool pdl_enabled() {
    if (g_pdl < 0) {
        const char* e = getenv("MRS_PDL");
        g_pdl = (e && e[0] == '1') ? 1 : 0;
    }
    return g_pdl == 1;
}

void set_pdl(int on) { g_pdl = on ? 1 : 0; }

// cudaLaunchKernelEx with programmatic stream serialization (PDL).
template <typename... KArgs, typename... Args>
static cudaError_t launch_ex(void (*kern)(KArgs...), int grid, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

// Resident CTAs per SM of a kernel (cached per function).
static int blocks_per_sm(const void* fn) {
    static std::mutex mu;
    static std::unordered_map<const void*, int> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(fn);
    if (it != cache.end()) return it->second;
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, kThreads, 0) != cudaSuccess || b < 1)
        b = 1;
    if (b > kMaxGridPerSM) b = kMaxGridPerSM;
    cache[fn] = b;
    return b;
}

// One wave: min(groups needed, resident CTAs); chunk = rows per CTA, a
// multiple of `rows_per_pass`.
static void wave_grid(const void* fn, int64_t nrows, int64_t rows_per_pass, int& grid,
                      int64_t& chunk) {
    const int64_t passes = (nrows + rows_per_pass - 1) / rows_per_pass;
    int64_t g = (int64_t)blocks_per_sm(fn) * num_sms();
    if (g > passes) g = passes;
    if (g < 1) g = 1;
    const int64_t per = (passes + g - 1) / g;
    chunk = per * rows_per_pass;
    grid = (int)((passes + per - 1) / per);
}

int spmm_grid(int64_t nrows, int64_t m) {   // upper bound (scratch sizing)
    (void)nrows; (void)m;
    return max_grid();
}

int vec_grid(int64_t n, int64_t m) {
    (void)n; (void)m;
    return max_grid();
}

// cudaLaunchKernelEx with dynamic shared memory (staged SpMM).
template <typename... KArgs, typename... Args>
static cudaError_t launch_ex_smem(void (*kern)(KArgs...), int grid, size_t smem, cudaStream_t s,
                                  Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

static int staged_blocks_per_sm(const void* fn, size_t smem) {
    static std::mutex mu;
    static std::unordered_map<const void*, int> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(fn);
    if (it != cache.end()) return it->second;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, kThreads, smem) != cudaSuccess || b < 1)
        b = 1;
    if (b > kMaxGridPerSM) b = kMaxGridPerSM;
    cache[fn] = b;
    return b;
}

template <int M, int OP, typename Tv, typename Ti>
static void launch_staged(SpArgs a, cudaStream_t s) {
    auto kern = spmm_staged_kernel<M, OP, Tv, Ti>;
    constexpr size_t smem = stage_bytes<Tv, Ti>();
    const int64_t rpp = Lay<M>::RPB;
    const int64_t cap = (int64_t)staged_blocks_per_sm((const void*)kern, smem) * num_sms();
    int64_t passes = a.nrows / (rpp * cap);
    const int64_t pmax = rpp >= 512 ? 1 : 512 / rpp;
    passes = passes < 1 ? 1 : (passes > pmax ? pmax : passes);
    a.chunk = rpp * passes;
    const int64_t nchunks = (a.nrows + a.chunk - 1) / a.chunk;
    int g = (int)(nchunks < cap ? nchunks : cap);
    if (g < 1) g = 1;
    (void)launch_ex_smem(kern, g, smem, s, a);
}

template <int OP, typename Tv, typename Ti>
static cudaError_t spmm_m(SpArgs a, int64_t m, cudaStream_t s, bool generic) {
    int g;
    if (g_staged && !generic) {
        switch (m) {
        case 1: launch_staged<1, OP, Tv, Ti>(a, s); return cudaGetLastError();
        case 2: launch_staged<2, OP, Tv, Ti>(a, s); return cudaGetLastError();
        case 4: launch_staged<4, OP, Tv, Ti>(a, s); return cudaGetLastError();
        case 8: launch_staged<8, OP, Tv, Ti>(a, s); return cudaGetLastError();
        case 16: launch_staged<16, OP, Tv, Ti>(a, s); return cudaGetLastError();
        case 32: launch_staged<32, OP, Tv, Ti>(a, s); return cudaGetLastError();
        case 64: launch_staged<64, OP, Tv, Ti>(a, s); return cudaGetLastError();
        default: break;
        }
    }
    auto go = [&](auto kern, int64_t rpp) {
        // chunks of up to ~512 rows (fewer when that would idle SMs), strided
        // over one wave of CTAs
        const int64_t cap = (int64_t)blocks_per_sm((const void*)kern) * num_sms();
        int64_t passes = a.nrows / (rpp * cap);
        const int64_t pmax = rpp >= 512 ? 1 : 512 / rpp;
        passes = passes < 1 ? 1 : (passes > pmax ? pmax : passes);
        const int64_t chunk = rpp * passes;
        const int64_t nchunks = (a.nrows + chunk - 1) / chunk;
        g = (int)(nchunks < cap ? nchunks : cap);
        if (g < 1) g = 1;
        a.chunk = chunk;
        (void)launch_ex(kern, g, s, a);
    };
    switch (generic ? 0 : m) {
    case 1: go(spmm_kernel<1, OP, Tv, Ti>, Lay<1>::RPB); break;
    case 2: go(spmm_kernel<2, OP, Tv, Ti>, Lay<2>::RPB); break;
    case 4: go(spmm_kernel<4, OP, Tv, Ti>, Lay<4>::RPB); break;
    case 8: go(spmm_kernel<8, OP, Tv, Ti>, Lay<8>::RPB); break;
    case 16: go(spmm_kernel<16, OP, Tv, Ti>, Lay<16>::RPB); break;
    case 32: go(spmm_kernel<32, OP, Tv, Ti>, Lay<32>::RPB); break;
    case 64: go(spmm_kernel<64, OP, Tv, Ti>, Lay<64>::RPB); break;
    default: go(spmm_kernel_generic<OP, Tv, Ti>, kThreads / m); break;
    }
    return cudaGetLastError();
}

template <int OP>
static cudaError_t spmm_op(const DevCsr& A, const SpArgs& a, int64_t m, cudaStream_t s, bool g) {
    if (A.vb == 8) {
        if (A.ib == 4) return spmm_m<OP, double, uint32_t>(a, m, s, g);
        if (A.ib == 2) return spmm_m<OP, double, uint16_t>(a, m, s, g);
        if constexpr (OP == OP_SPMV)
            if (A.ib == 1) return spmm_m<OP, double, uint8_t>(a, m, s, g);
    } else if (A.vb == 4) {
        if (A.ib == 4) return spmm_m<OP, float, uint32_t>(a, m, s, g);
        if (A.ib == 2) return spmm_m<OP, float, uint16_t>(a, m, s, g);
        if constexpr (OP == OP_SPMV)
            if (A.ib == 1) return spmm_m<OP, float, uint8_t>(a, m, s, g);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_spmm(int op, const DevCsr& A, SpArgs a, int64_t m, cudaStream_t s,
                        bool generic) {
    a.rp = A.rp; a.ci = A.ci; a.vals = A.v; a.nrows = A.nrows; a.m = m;
    if (A.nrows == 0) return cudaSuccess;
    switch (op) {
    case OP_SPMV: return spmm_op<OP_SPMV>(A, a, m, s, generic);
    case OP_JAC_SWEEP: return spmm_op<OP_JAC_SWEEP>(A, a, m, s, generic);
    case OP_CHEB_FIRST: return spmm_op<OP_CHEB_FIRST>(A, a, m, s, generic);
    case OP_CHEB_STEP: return spmm_op<OP_CHEB_STEP>(A, a, m, s, generic);
    }
    return cudaErrorInvalidValue;
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
    }
    return cudaErrorInvalidValue;
}

// Coarsest level: x = Ainv b (replaces scipy lu_solve, solvers.py:644-649).
// CTA handles kRows rows; thread (ks, c) folds k = ks, ks + kpb, ... for
// column c, then the ks partials are folded in order (deterministic).
constexpr int kCoarseRows = 4;

__global__ void __launch_bounds__(kThreads) coarse_kernel(const double* __restrict__ inv, int64_t nc,
                                                          const double* __restrict__ b,
                                                          double* __restrict__ x, int m,
                                                          const int* guard) {
    pdl_enter();
    if (guard && *guard) return;
    __shared__ double s_t[kThreads];
    const int kpb = kThreads / m;
    const int c = threadIdx.x % m, ks = threadIdx.x / m;
    for (int rr = 0; rr < kCoarseRows; ++rr) {
        int64_t i = (int64_t)blockIdx.x * kCoarseRows + rr;
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
    int g = (int)((nc + kCoarseRows - 1) / kCoarseRows);
    (void)launch_ex(coarse_kernel, g, s, inv, nc, b, x, (int)m, guard);
    return cudaGetLastError();
}

}  // namespace mrs
