// launch.cuh -- launch helpers shared by the kernel translation units
// (occupancy-sized one-wave grids, PDL launch attribute).
#pragma once

#include <algorithm>
#include <mutex>
#include <unordered_map>

#include "dispatch.h"

namespace mrs {

int64_t spmm_long_max_rows();   // LONG-row SpMM variant up to this many rows (knob)
int64_t spmm_chunk_rows();      // rows per CTA chunk of the SpMM grid (knob)
int64_t spmm_coop();            // cooperative entry loads for long-row operators (knob)
int64_t spmm_variant();         // force one SpmmVariant everywhere (knob; 0 = per operator)
int64_t spmm_pair();            // pair loads for long-row operators (knob)


// cudaLaunchKernelEx with programmatic stream serialization (PDL).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_ex_smem(void (*kern)(KArgs...), int grid, size_t smem, cudaStream_t s,
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

template <typename... KArgs, typename... Args>
inline cudaError_t launch_ex(void (*kern)(KArgs...), int grid, cudaStream_t s, Args... args) {
    return launch_ex_smem(kern, grid, 0, s, args...);
}

// Resident CTAs per SM of a kernel (cached per function).
inline int blocks_per_sm(const void* fn, size_t smem = 0) {
    static std::mutex mu;
    static std::unordered_map<const void*, int> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(fn);
    if (it != cache.end()) return it->second;
    int b = 0;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, kThreads, smem) != cudaSuccess || b < 1)
        b = 1;
    if (b > kMaxGridPerSM) b = kMaxGridPerSM;
    cache[fn] = b;
    return b;
}

// One wave: min(groups needed, resident CTAs); chunk = rows per CTA, a
// multiple of `rows_per_pass`.
inline void wave_grid(const void* fn, int64_t nrows, int64_t rows_per_pass, int& grid,
                      int64_t& chunk) {
    const int64_t passes = (nrows + rows_per_pass - 1) / rows_per_pass;
    int64_t g = (int64_t)blocks_per_sm(fn) * num_sms();
    if (g > passes) g = passes;
    if (g < 1) g = 1;
    const int64_t per = (passes + g - 1) / g;
    chunk = per * rows_per_pass;
    grid = (int)((passes + per - 1) / per);
}


// SV_PAIR (round 2): large operators with >= 12 entries per row fetch their entries
// as aligned pairs -- knob spmm_pair: 1 instead of LANE, 2 (default) also instead of
// COOP (whose shuffles run on the same L1 data pipe as the loads they save).
// Whole-solve A/B (profiles/r02s4_pair_variant.txt): C3 60.3 -> 58.6 ms, C4 53.8 -> 51.6 ms.
// Shape heuristic (the default when an operator carries no measured choice):
// small operators with long rows -> LONG (16 entries in flight); large
// operators with long AND uniform rows (27-point stencils: mean >= 20, no row
// more than ~10 % above it) -> COOP (knob spmm_coop: 1 = every operator with
// >= 12 entries per row); otherwise LANE.  Set by hand on whole solves in
// round 1 (profiles/r01_ab_experiments.txt).
inline int spmm_shape_variant(int64_t nr, int64_t nnz, int max_row, int64_t m) {
    const int64_t coop = spmm_coop();
    const bool uniform_long = nnz >= 20 * nr && max_row > 0 &&
                              (int64_t)max_row * 10 * nr <= 11 * nnz + 10 * nr;
    if (m <= 16 && nr <= spmm_long_max_rows() && nnz >= 12 * nr) return SV_LONG;
    const int64_t pair = spmm_pair();
    // (operators under ~200 k rows are latency-bound, not L1-pipe-bound: the pair
    // kernel's peeling costs them ~1 %, measured on C2's level 1)
    const bool pair_ok = (m == 2 || m == 4 || m == 8 || m == 16) && nnz >= 12 * nr &&
                         nr >= 200000;
    if ((m == 4 || m == 8 || m == 16) &&
        ((coop == 1 && nnz >= 12 * nr) || (coop == 2 && uniform_long)))
        return (pair == 2 && pair_ok) ? SV_PAIR : SV_COOP;
    if (pair >= 1 && pair_ok) return SV_PAIR;
    return SV_LANE;
}

// SpMM family: chunk-strided one-wave grid (see spmm.cuh).  Tx / Ty: vector
// types (double, or the float levels of the fp32-vector V-cycle: lane and
// LONG variants, m in {1, 2, 4, 8, 16, 32}).
template <int OP, typename Tv, typename Ti, typename Tx = double, typename Ty = double>
inline cudaError_t spmm_m(SpArgs a, int64_t m, cudaStream_t s, bool generic) {
    constexpr bool kF64 = sizeof(Tx) == 8 && sizeof(Ty) == 8;
    int g;
    auto go = [&](auto kern, int64_t rpp) {
        // Balanced one wave: every CTA gets the same number of passes (the
        // slowest CTA sets the kernel time), in chunks of ~64 rows strided
        // over the grid: the active band of the matrix stays narrow (grid x 64
        // rows), so gathered x rows shared by rows a plane apart are still in
        // L2 when the later row reads them (scripts/probe/spmm_probe.cu:
        // 512-row chunks 244 -> 64-row chunks 207 us on the 128^3 m=16 SpMM).
        const int64_t cap = (int64_t)blocks_per_sm((const void*)kern) * num_sms();
        const int64_t P = (a.nrows + rpp - 1) / rpp;             // passes in total
        const int64_t ppc = (P + cap - 1) / cap;                  // passes per CTA
        const int64_t pmax = rpp >= spmm_chunk_rows() ? 1 : spmm_chunk_rows() / rpp;
        const int64_t sp = ppc < pmax ? ppc : pmax;               // passes per chunk
        const int64_t nchunks = (P + sp - 1) / sp;
        const int64_t cpc = (nchunks + cap - 1) / cap;            // chunks per CTA
        g = (int)((nchunks + cpc - 1) / cpc);
        if (g < 1) g = 1;
        a.chunk = rpp * sp;
        if (generic) a.n_long = 0;                               // lane path only
        a.long_ctas = (a.n_long && !a.no_long_ctas)
                          ? (int)std::min<int64_t>(a.n_long, 4LL * num_sms()) : 0;
        (void)launch_ex_smem(kern, g + a.long_ctas,
                             a.long_ctas ? kLongProducts * sizeof(double) : 0, s, a);
    };
    int v = a.variant ? a.variant : (int)spmm_variant();
    if (v == SV_AUTO)
        v = spmm_shape_variant(a.rows_hint, a.nnz_hint, a.max_row_hint, m);
    // pair loads need naturally aligned entry arrays (cudaMalloc'ed ones are)
    if (v == SV_PAIR && (((uintptr_t)a.vals & 15u) || ((uintptr_t)a.ci & 15u))) v = SV_LANE;
    if (!generic && v == SV_LONG) {
        switch (m) {
        case 1: go(spmm_kernel<1, OP, Tv, Ti, true, false, Tx, Ty>, Lay<1>::RPB); return cudaGetLastError();
        case 2: go(spmm_kernel<2, OP, Tv, Ti, true, false, Tx, Ty>, Lay<2>::RPB); return cudaGetLastError();
        case 4: go(spmm_kernel<4, OP, Tv, Ti, true, false, Tx, Ty>, Lay<4>::RPB); return cudaGetLastError();
        case 8: go(spmm_kernel<8, OP, Tv, Ti, true, false, Tx, Ty>, Lay<8>::RPB); return cudaGetLastError();
        case 16: go(spmm_kernel<16, OP, Tv, Ti, true, false, Tx, Ty>, Lay<16>::RPB); return cudaGetLastError();
        default: break;
        }
    }
    if (!generic && v == SV_PAIR) {          // any vector precision
        switch (m) {
        case 2: go(spmm_kernel<2, OP, Tv, Ti, false, false, Tx, Ty, 3>, Lay<2>::RPB); return cudaGetLastError();
        case 4: go(spmm_kernel<4, OP, Tv, Ti, false, false, Tx, Ty, 3>, Lay<4>::RPB); return cudaGetLastError();
        case 8: go(spmm_kernel<8, OP, Tv, Ti, false, false, Tx, Ty, 3>, Lay<8>::RPB); return cudaGetLastError();
        case 16: go(spmm_kernel<16, OP, Tv, Ti, false, false, Tx, Ty, 3>, Lay<16>::RPB); return cudaGetLastError();
        default: break;
        }
    }
    if constexpr (kF64) {
        if (!generic && (v == SV_LANE_L2 || v == SV_LANE_NA)) {
            const bool l2 = v == SV_LANE_L2;
            switch (m) {
            case 1: l2 ? go(spmm_kernel<1, OP, Tv, Ti, false, false, double, double, 1>, Lay<1>::RPB)
                       : go(spmm_kernel<1, OP, Tv, Ti, false, false, double, double, 2>, Lay<1>::RPB);
                return cudaGetLastError();
            case 2: l2 ? go(spmm_kernel<2, OP, Tv, Ti, false, false, double, double, 1>, Lay<2>::RPB)
                       : go(spmm_kernel<2, OP, Tv, Ti, false, false, double, double, 2>, Lay<2>::RPB);
                return cudaGetLastError();
            case 4: l2 ? go(spmm_kernel<4, OP, Tv, Ti, false, false, double, double, 1>, Lay<4>::RPB)
                       : go(spmm_kernel<4, OP, Tv, Ti, false, false, double, double, 2>, Lay<4>::RPB);
                return cudaGetLastError();
            case 8: l2 ? go(spmm_kernel<8, OP, Tv, Ti, false, false, double, double, 1>, Lay<8>::RPB)
                       : go(spmm_kernel<8, OP, Tv, Ti, false, false, double, double, 2>, Lay<8>::RPB);
                return cudaGetLastError();
            case 16: l2 ? go(spmm_kernel<16, OP, Tv, Ti, false, false, double, double, 1>, Lay<16>::RPB)
                        : go(spmm_kernel<16, OP, Tv, Ti, false, false, double, double, 2>, Lay<16>::RPB);
                return cudaGetLastError();
            default: break;
            }
        }
        if (!generic && v == SV_COOP) {
            switch (m) {
            case 4: go(spmm_kernel<4, OP, Tv, Ti, false, true>, Lay<4>::RPB); return cudaGetLastError();
            case 8: go(spmm_kernel<8, OP, Tv, Ti, false, true>, Lay<8>::RPB); return cudaGetLastError();
            case 16: go(spmm_kernel<16, OP, Tv, Ti, false, true>, Lay<16>::RPB); return cudaGetLastError();
            default: break;
            }
        }
    }
    switch (generic ? 0 : m) {
    case 1: go(spmm_kernel<1, OP, Tv, Ti, false, false, Tx, Ty>, Lay<1>::RPB); break;
    case 2: go(spmm_kernel<2, OP, Tv, Ti, false, false, Tx, Ty>, Lay<2>::RPB); break;
    case 4: go(spmm_kernel<4, OP, Tv, Ti, false, false, Tx, Ty>, Lay<4>::RPB); break;
    case 8: go(spmm_kernel<8, OP, Tv, Ti, false, false, Tx, Ty>, Lay<8>::RPB); break;
    case 16: go(spmm_kernel<16, OP, Tv, Ti, false, false, Tx, Ty>, Lay<16>::RPB); break;
    case 32: go(spmm_kernel<32, OP, Tv, Ti, false, false, Tx, Ty>, Lay<32>::RPB); break;
    default:
        if constexpr (kF64) {
            if (!generic && m == 64) go(spmm_kernel<64, OP, Tv, Ti>, Lay<64>::RPB);
            else go(spmm_kernel_generic<OP, Tv, Ti>, kThreads / m);
        } else {
            return cudaErrorInvalidValue;     // float vectors: m in {1, ..., 32} powers of 2
        }
        break;
    }
    return cudaGetLastError();
}

// Vector precision of one launch (SpArgs::vp): VP_DD all double; VP_FF all
// float (a float level); VP_DF double gathered operand -> float row operands
// (restriction into a float level); VP_FD float gathered -> double row
// operands (prolongation from a float level).
template <int OP, typename Tv, typename Ti>
inline cudaError_t spmm_vp(const SpArgs& a, int64_t m, cudaStream_t s, bool g) {
    switch (a.vp) {
    case VP_DD: return spmm_m<OP, Tv, Ti>(a, m, s, g);
    case VP_FF: return spmm_m<OP, Tv, Ti, float, float>(a, m, s, g);
    case VP_DF:
        if constexpr (OP == OP_SPMV) return spmm_m<OP, Tv, Ti, double, float>(a, m, s, g);
        break;
    case VP_FD:
        if constexpr (OP == OP_SPMV) return spmm_m<OP, Tv, Ti, float, double>(a, m, s, g);
        break;
    }
    return cudaErrorInvalidValue;
}

template <int OP, typename Tv>
inline cudaError_t spmm_op(const DevCsr& A, const SpArgs& a, int64_t m, cudaStream_t s, bool g) {
    if (A.ib == 4) return spmm_vp<OP, Tv, uint32_t>(a, m, s, g);
    if (A.ib == 2) return spmm_vp<OP, Tv, uint16_t>(a, m, s, g);
    if constexpr (OP == OP_SPMV)
        if (A.ib == 1) return spmm_m<OP, Tv, uint8_t>(a, m, s, g);     // plugin: double only
    return cudaErrorInvalidValue;
}

// One translation unit per (value type, op) (spmm_<t>_<op>.cu): parallel builds.
template <int OP>
cudaError_t launch_spmm_op_f64(const DevCsr& A, const SpArgs& a, int64_t m, cudaStream_t s,
                               bool generic);
template <int OP>
cudaError_t launch_spmm_op_f32(const DevCsr& A, const SpArgs& a, int64_t m, cudaStream_t s,
                               bool generic);

}  // namespace mrs
