// spmm.cuh -- multi-RHS CSR SpMM engine and its fused smoother variants.
//
// Replaces the reference's `csr_spmv` (_ckernels.pyx:30-57) and the numpy
// updates that follow it in the smoothers (blas2.py:176-181 Jacobi,
// solvers.py:545-571 Chebyshev).
//
// Layout: the m right-hand sides of one row are contiguous (row-major (n, m)
// block).  A row is owned by a group of LPR = M / CPL lanes; lane l owns the
// CPL consecutive columns [l*CPL, (l+1)*CPL) and moves them with 16-byte
// vector loads/stores, so a warp touches 32*CPL*8 contiguous bytes of y and
// LPR*CPL*8 contiguous bytes of each gathered x row.  Each (row, column) is
// accumulated sequentially in CSR entry order with separately rounded
// mul/add, i.e. bitwise the reference kernel.
//
//   M   : 1  2  4  8  16  32  64   (0 = any m, generic path)
//   CPL : 1  2  2  2   2   4   8
//   LPR : 1  1  2  4   8   8   8
//
// Grid: one wave of resident CTAs (occupancy-sized, never more than the rows
// need) striding over chunks of ~64 consecutive rows.  Inside a chunk the
// CTA walks passes of RPB rows, so x rows shared by neighbouring passes are
// reused from L1; across CTAs the active chunks form one narrow band of the
// matrix, so the gathered x window of a banded matrix stays L2-resident.
// The reduction shape of the fused dots is fixed by (n, grid): deterministic.
// Rows much longer than the operator's mean (AMG coarse levels) are taken
// out of the lane path and done by trailing CTAs, one row each
// (long_row_cta), so one long row no longer sets the kernel's duration.
#pragma once

#include "reduce.cuh"

namespace mrs {

template <int M> struct Lay {
    static constexpr int CPL = (M == 1) ? 1 : (M <= 16 ? 2 : M / 8);
    static constexpr int LPR = M / CPL;
    static constexpr int RPB = kThreads / LPR;     // rows per CTA pass
    static constexpr int UNR = 4;                  // entries in flight per lane
};

// Lane-path variants of one SpMM (all bitwise identical; per-operator choice,
// csrc/solver.cu autotune / knob spmm_variant).
enum SpmmVariant : int {
    SV_AUTO = 0,     // shape heuristic (launch.cuh spmm_m)
    SV_LANE = 1,     // LPR lanes per row, every lane loads every entry, 4 in flight
    SV_COOP = 2,     // lanes load distinct entries and shuffle (m in {4, 8, 16})
    SV_LONG = 3,     // 16 entries in flight per lane, 1 CTA/SM (m <= 16)
    SV_LANE_L2 = 4,  // lane, gathered x through L2 only (ld.global.cg: no L1 fills)
    SV_LANE_NA = 5,  // lane, gathered x with L1::no_allocate (hits kept, misses not filled)
    SV_STREAM = 6,   // m = 1, banded operators: TMA-fed entry-parallel products (stream.cu)
    SV_PAIR = 7,     // lane, entries loaded as aligned PAIRS (one 16-byte value load and one
                     // 4/8-byte index load per two entries): half the L1 wavefronts of the
                     // matrix stream on long-row operators (a warp's 8 rows sit in 8 lines)
};

// Vector precisions of one SpMM launch (gathered operand -> row operands).
enum VecPrec : int { VP_DD = 0, VP_FF = 1, VP_DF = 2, VP_FD = 3 };

// Kernel operation selector.
enum SpOp : int {
    OP_SPMV = 0,         // y op= A x by `mode` (+ optional next-level seed)   (csr_spmv)
    OP_JAC_SWEEP,        // x' = x + w*((b - A x)/d)                           (jacobi_sweep)
    OP_CHEB_FIRST,       // r = b - A x; dv = r/(d*theta); x' = x + dv          (chebyshev first step)
    OP_CHEB_STEP,        // tmp = A dv; r -= tmp; dv' = dv*c1 + c2*(r/d); x += dv'
};
// Zero-guess first steps never gather on-the-fly values: the producer of a
// level's right-hand side emits the seed (see SpArgs::seed, VArgs::seed).

struct SpArgs {
    const int32_t* rp;
    const void* ci;
    const void* vals;
    int64_t nrows;
    int64_t m;              // runtime m (generic path / strides)
    const double* x;        // gathered operand (x or dv)
    const double* b;        // right-hand side (RSUB / smoothers)
    const double* d;        // diagonal (smoothers)
    double* y;              // OP_SPMV output
    const double* x_in;     // own-row x (cheb step)
    const double* r_in;     // own-row r (cheb step)
    double* x_out;
    double* r_out;
    double* dv_out;
    double w, theta, c1, c2;
    int mode;
    const int* guard;       // non-null: skip the kernel when *guard != 0
    int dot;                // fused per-column dot: OP_SPMV x_own.y_out;
                            // smoother ops b_own.x_new (PCG's (r, z))
    int seed;               // OP_SPMV (restriction): also emit the next level's
                            // zero-guess smoother seed from the row result:
                            // 1: seed_out = w*(y/d)  2: seed_out = y/(d*theta)
    double* seed_out;
    int64_t chunk;          // rows per CTA (contiguous range, multiple of RPB)
    int64_t nnz_hint;       // matrix nnz (layout choice)
    const int32_t* slab_base;  // non-null: column = slab_base[row >> slab_shift] + col16
    int slab_shift;
    int64_t ncols_hint;     // matrix columns
    const int32_t* long_rows;  // rows with more than long_thr entries (one CTA each)
    int n_long, long_thr, long_ctas;   // long_ctas: trailing CTAs of the grid doing them
    int max_row_hint;          // longest row (0: unknown) -- layout choice
    // row range of a split launch (multi-GPU halo overlap): rows
    // [row0, row0 + vrows) (vrows 0 = every row).  HOST-side only: the
    // launcher offsets every row-indexed pointer by row0 and the kernel walks
    // rows 0 .. vrows-1 -- a row offset inside the kernel's loop (even only in
    // its bounds) measured 9-10 % slower on the 7-point SpMM.  xo: the
    // gathered operand's own-row view (x + row0 * m; = x when unsplit).
    // no_long_ctas: this launch leaves the long rows to another launch.
    int64_t row0;
    int no_long_ctas;
    int64_t vrows;
    const double* xo;
    int64_t rows_hint;      // the operator's row count (variant choice)
    int variant;            // SpmmVariant forced for this operator (0 = heuristic)
    int vp;                 // vector precision (VP_*: fp32-vector V-cycle levels)
    RedArgs red;
};

// shared-memory products per chunk of a long row (long_row_cta)
constexpr int kLongProducts = 2048;

// Zero-guess smoother seed of a right-hand-side value v at a row with
// diagonal d: Jacobi's first sweep x = 0 + w*(v/d) (blas2.py:181) or
// Chebyshev's first step dv = v/(d*theta) (solvers.py:551).
// Mode 3: Gauss-Seidel starts from x = 0 (no shortcut): the seed is 0.
__device__ __forceinline__ double seed_value(int mode, double v, double d, double w_or_theta) {
    if (mode == 3) return 0.0;
    return mode == 1 ? mul(w_or_theta, divd(v, d)) : divd(v, mul(d, w_or_theta));
}

// Typed vector operands.  Each level's block vectors are double, or float in
// the fp32-vector V-cycle (plan option vec32): loads widen to double, stores
// round to the vector's type; accumulation is always double.  Tx = type of the
// gathered operand (x / dv), Ty = type of the row operands (b, y, seed, x_out,
// r, dv ...).  Transfers between a double and a float level mix the two.
template <int CPL, typename T>
__device__ __forceinline__ Vec<CPL> ldt(const T* p) {        // read-only path
    if constexpr (sizeof(T) == 8) {
        return load_vec<CPL>(reinterpret_cast<const double*>(p));
    } else {
        Vec<CPL> r;
        if constexpr (CPL == 1) {
            r.v[0] = (double)__ldg(p);
        } else if constexpr (CPL == 2) {
            const float2 t = __ldg(reinterpret_cast<const float2*>(p));
            r.v[0] = t.x; r.v[1] = t.y;
        } else {
#pragma unroll
            for (int i = 0; i < CPL; i += 4) {
                const float4 t = __ldg(reinterpret_cast<const float4*>(p + i));
                r.v[i] = t.x; r.v[i + 1] = t.y; r.v[i + 2] = t.z; r.v[i + 3] = t.w;
            }
        }
        return r;
    }
}
template <int CPL, typename T>
__device__ __forceinline__ Vec<CPL> ldt_rw(const T* p) {     // coherent (read-modify-write)
    if constexpr (sizeof(T) == 8) {
        return load_vec_rw<CPL>(reinterpret_cast<const double*>(p));
    } else {
        Vec<CPL> r;
        if constexpr (CPL == 1) {
            r.v[0] = (double)*p;
        } else if constexpr (CPL == 2) {
            const float2 t = *reinterpret_cast<const float2*>(p);
            r.v[0] = t.x; r.v[1] = t.y;
        } else {
#pragma unroll
            for (int i = 0; i < CPL; i += 4) {
                const float4 t = *reinterpret_cast<const float4*>(p + i);
                r.v[i] = t.x; r.v[i + 1] = t.y; r.v[i + 2] = t.z; r.v[i + 3] = t.w;
            }
        }
        return r;
    }
}
template <int CPL, typename T>
__device__ __forceinline__ void stt(T* p, const Vec<CPL>& a) {
    if constexpr (sizeof(T) == 8) {
        store_vec<CPL>(reinterpret_cast<double*>(p), a);
    } else if constexpr (CPL == 1) {
        *p = __double2float_rn(a.v[0]);
    } else if constexpr (CPL == 2) {
        *reinterpret_cast<float2*>(p) = make_float2(__double2float_rn(a.v[0]),
                                                    __double2float_rn(a.v[1]));
    } else {
#pragma unroll
        for (int i = 0; i < CPL; i += 4)
            *reinterpret_cast<float4*>(p + i) =
                make_float4(__double2float_rn(a.v[i]), __double2float_rn(a.v[i + 1]),
                            __double2float_rn(a.v[i + 2]), __double2float_rn(a.v[i + 3]));
    }
}
// typed views of the SpArgs operand pointers (declared double*; a float
// level's buffers are passed through them)
template <typename T> __device__ __forceinline__ const T* tp(const double* p) {
    return reinterpret_cast<const T*>(p);
}
template <typename T> __device__ __forceinline__ T* tpw(double* p) {
    return reinterpret_cast<T*>(p);
}

// Value of the gathered operand at column `col` (CPL columns at cofs).
// LM: cache mode of the gathered operand (double only): 0 read-only path,
// 1 L2 only (cg), 2 L1 no-allocate.  Operators whose gathers rarely hit L1
// (random columns over a window larger than L1, e.g. the C5 band) spend the
// L1 data pipe on fills that are never reused; the choice is measured per
// operator (SpmmVariant SV_LANE_L2 / SV_LANE_NA).
__device__ __forceinline__ double2 ld_na2(const double* p) {
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
                 : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ double ld_na1(const double* p) {
    double r;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
    return r;
}
template <int CPL, int LM>
__device__ __forceinline__ Vec<CPL> ld_mode(const double* p) {
    if constexpr (LM == 0) return load_vec<CPL>(p);
    Vec<CPL> r;
    if constexpr (CPL == 1) {
        r.v[0] = LM == 1 ? __ldcg(p) : ld_na1(p);
    } else {
#pragma unroll
        for (int i = 0; i < CPL; i += 2) {
            const double2 t = LM == 1 ? __ldcg(reinterpret_cast<const double2*>(p + i))
                                      : ld_na2(p + i);
            r.v[i] = t.x; r.v[i + 1] = t.y;
        }
    }
    return r;
}

template <int CPL, typename Tx, int LM = 0>
__device__ __forceinline__ Vec<CPL> gather(const SpArgs& a, int col, int ld, int cofs) {
    if constexpr (sizeof(Tx) == 8 && LM != 0) return ld_mode<CPL, LM>(a.x + col * ld + cofs);
    else return ldt<CPL>(tp<Tx>(a.x) + col * ld + cofs);
}

// Where a row's (column, value) entries come from (global memory, read-only
// path); slab-compressed indices add the row's slab base.
template <typename Tv, typename Ti> struct GSrc {
    const Ti* __restrict__ ci;
    const Tv* __restrict__ v;
    int base = 0;          // slab-compressed indices: column = base(row) + ci
    __device__ __forceinline__ int col(int k) const {
        const int c = base + (int)__ldg(ci + k);
        MRS_DCHECK(c >= 0);
        return c;
    }
    __device__ __forceinline__ double val(int k) const { return widen(__ldg(v + k)); }
    // entries k, k + 1 with ONE value load and ONE index load (k even: the arrays
    // are 16-byte aligned, so the pair is naturally aligned)
    __device__ __forceinline__ void pair(int k, int& c0, int& c1, double& v0, double& v1) const {
        if constexpr (sizeof(Tv) == 8) {
            const double2 t = __ldg(reinterpret_cast<const double2*>(v + k));
            v0 = t.x; v1 = t.y;
        } else {
            const float2 t = __ldg(reinterpret_cast<const float2*>(v + k));
            v0 = (double)t.x; v1 = (double)t.y;
        }
        if constexpr (sizeof(Ti) == 4) {
            const uint2 w = __ldg(reinterpret_cast<const uint2*>(ci + k));
            c0 = base + (int)w.x; c1 = base + (int)w.y;
        } else if constexpr (sizeof(Ti) == 2) {
            const uint32_t w = __ldg(reinterpret_cast<const uint32_t*>(ci + k));
            c0 = base + (int)(w & 0xffffu); c1 = base + (int)(w >> 16);
        } else {
            const uint16_t w = __ldg(reinterpret_cast<const uint16_t*>(ci + k));
            c0 = base + (int)(w & 0xffu); c1 = base + (int)(w >> 8);
        }
        MRS_DCHECK(c0 >= 0 && c1 >= 0);
    }
    // the row's view: slab base of `row` (16-bit slab-relative columns)
    __device__ __forceinline__ GSrc at_row(const SpArgs& a, int row) const {
        GSrc r = *this;
        if (a.slab_base) r.base = __ldg(a.slab_base + (row >> a.slab_shift));
        return r;
    }
};

// Accumulate one row: acc op= sum_k v_k * g(col_k), entry order; the loads
// of a group of UNR entries are issued before their (ordered) accumulation.
template <int CPL, bool SUBTRACT, typename Tx, class Src, int UNR = 4, int LM = 0>
__device__ __forceinline__ void row_accumulate(const SpArgs& a, const Src& src, int lo,
                                               int hi, int ld, int cofs,
                                               double (&acc)[CPL]) {
    // Entries in groups of UNR: all loads of a group are issued before the
    // group is accumulated in entry order.  The last, partial group loads
    // entry `lo` in its empty slots (valid addresses, no branches) and only
    // accumulates its live entries: a 7-entry row costs two dependent load
    // rounds instead of 1 + 3.
    const int klo = (int)lo, khi = (int)hi;
    for (int k = klo; k < khi; k += UNR) {
        int c[UNR];
        double v[UNR];
        Vec<CPL> g[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const int kk = (k + u < khi) ? k + u : klo;
            c[u] = (int)src.col(kk);
            v[u] = src.val(kk);
        }
        compiler_fence();   // keep the group's loads issued together (the
                            // scheduler otherwise interleaves them with uses)
#pragma unroll
        for (int u = 0; u < UNR; ++u) g[u] = gather<CPL, Tx, LM>(a, c[u], ld, cofs);
        compiler_fence();
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            if (k + u < khi) {
#pragma unroll
                for (int i = 0; i < CPL; ++i) {
                    if constexpr (SUBTRACT) acc[i] = sub(acc[i], mul(v[u], g[u].v[i]));
                    else acc[i] = add(acc[i], mul(v[u], g[u].v[i]));
                }
            }
        }
    }
}

// SV_PAIR: the same entry order, entries fetched as aligned pairs (LM == 3).
template <int CPL, bool SUBTRACT, typename Tx, class Src>
__device__ __forceinline__ void row_accumulate_pairs(const SpArgs& a, const Src& src, int lo, int hi,
                                                     int ld, int cofs, double (&acc)[CPL]) {
    auto fma1 = [&](double v, const Vec<CPL>& g) {
#pragma unroll
        for (int i = 0; i < CPL; ++i) {
            if constexpr (SUBTRACT) acc[i] = sub(acc[i], mul(v, g.v[i]));
            else acc[i] = add(acc[i], mul(v, g.v[i]));
        }
    };
    int k = lo;
    if ((k & 1) && k < hi) {                         // odd first entry: alone
        const int c = src.col(k);
        const double v = src.val(k);
        fma1(v, gather<CPL, Tx, 0>(a, c, ld, cofs));
        ++k;
    }
    for (; k + 3 < hi; k += 4) {                     // two pairs in flight
        int c[4];
        double v[4];
        Vec<CPL> g[4];
        src.pair(k, c[0], c[1], v[0], v[1]);
        src.pair(k + 2, c[2], c[3], v[2], v[3]);
        compiler_fence();
#pragma unroll
        for (int u = 0; u < 4; ++u) g[u] = gather<CPL, Tx, 0>(a, c[u], ld, cofs);
        compiler_fence();
#pragma unroll
        for (int u = 0; u < 4; ++u) fma1(v[u], g[u]);
    }
    if (k + 1 < hi) {
        int c0, c1;
        double v0, v1;
        src.pair(k, c0, c1, v0, v1);
        const Vec<CPL> g0 = gather<CPL, Tx, 0>(a, c0, ld, cofs);
        const Vec<CPL> g1 = gather<CPL, Tx, 0>(a, c1, ld, cofs);
        fma1(v0, g0);
        fma1(v1, g1);
        k += 2;
    }
    if (k < hi) {
        const int c = src.col(k);
        const double v = src.val(k);
        fma1(v, gather<CPL, Tx, 0>(a, c, ld, cofs));
    }
}

// One (row, column-slice) of work for every op, in three parts so that the
// long-row path (long_row_cta) can run the same prologue / epilogue around a
// CTA-cooperative accumulation.  row_begin loads the accumulator's start
// value; `subtract` = entries are subtracted.
template <int OP, int CPL, typename Ty>
__device__ __forceinline__ void row_begin(const SpArgs& a, int o, double (&acc)[CPL],
                                          bool& subtract) {
    if constexpr (OP == OP_SPMV) {
        const int mode = a.mode;
        if (mode == MRS_MODE_ASSIGN) {
#pragma unroll
            for (int i = 0; i < CPL; ++i) acc[i] = 0.0;
        } else if (mode == MRS_MODE_RSUB) {
            Vec<CPL> t = ldt<CPL>(tp<Ty>(a.b) + o);
#pragma unroll
            for (int i = 0; i < CPL; ++i) acc[i] = t.v[i];
        } else {
            Vec<CPL> t = ldt_rw<CPL>(tp<Ty>(a.y) + o);
#pragma unroll
            for (int i = 0; i < CPL; ++i) acc[i] = t.v[i];
        }
        subtract = !(mode == MRS_MODE_ASSIGN || mode == MRS_MODE_ADD);
    } else if constexpr (OP == OP_JAC_SWEEP || OP == OP_CHEB_FIRST) {
        // r = b - A x  (RSUB order: start at b, subtract in entry order); b
        // is re-read by row_end for the fused dot rather than held across
        // the accumulation (4 fewer live registers in the gather loop)
        Vec<CPL> bb = ldt<CPL>(tp<Ty>(a.b) + o);
#pragma unroll
        for (int i = 0; i < CPL; ++i) acc[i] = bb.v[i];
        subtract = true;
    } else {  // OP_CHEB_STEP: tmp = A dv from 0
#pragma unroll
        for (int i = 0; i < CPL; ++i) acc[i] = 0.0;
        subtract = false;
    }
}

// Fused dots exist only on double vectors (the Krylov level).
template <int OP, int CPL, typename Tx, typename Ty>
__device__ __forceinline__ void row_end(const SpArgs& a, int row, int o, double (&acc)[CPL],
                                        double (&dotp)[CPL]) {
    constexpr bool kDot = sizeof(Tx) == 8 && sizeof(Ty) == 8;
    if constexpr (OP == OP_SPMV) {
        Vec<CPL> out;
#pragma unroll
        for (int i = 0; i < CPL; ++i) out.v[i] = acc[i];
        stt<CPL>(tpw<Ty>(a.y) + o, out);
        if (a.seed) {
            const double dd = __ldg(a.d + row);
            const double wt = a.seed == 1 ? a.w : a.theta;
#pragma unroll
            for (int i = 0; i < CPL; ++i) out.v[i] = seed_value(a.seed, acc[i], dd, wt);
            stt<CPL>(tpw<Ty>(a.seed_out) + o, out);
        }
        if constexpr (kDot) {
            if (a.dot) {   // (x_in ? x_in : x)_own . y  (x_in: e.g. BiCGStab's r0)
                Vec<CPL> xo = ldt<CPL>((a.x_in ? a.x_in : a.xo) + o);
#pragma unroll
                for (int i = 0; i < CPL; ++i) dotp[i] = add(dotp[i], mul(xo.v[i], acc[i]));
            }
        }
    } else if constexpr (OP == OP_JAC_SWEEP || OP == OP_CHEB_FIRST) {
        const double dd = __ldg(a.d + row);
        Vec<CPL> xo = ldt<CPL>(tp<Ty>(a.xo) + o);
        if constexpr (OP == OP_CHEB_FIRST) {
            const double dt = mul(dd, a.theta);
            Vec<CPL> r, dv;
#pragma unroll
            for (int i = 0; i < CPL; ++i) {
                r.v[i] = acc[i];
                dv.v[i] = divd(acc[i], dt);                 // dv = r / (d*theta)
                xo.v[i] = add(xo.v[i], dv.v[i]);            // x + dv
            }
            if (a.r_out) stt<CPL>(tpw<Ty>(a.r_out) + o, r);
            if (a.dv_out) stt<CPL>(tpw<Ty>(a.dv_out) + o, dv);
        } else {
#pragma unroll
            for (int i = 0; i < CPL; ++i) xo.v[i] = add(xo.v[i], mul(a.w, divd(acc[i], dd)));  // blas2.py:181
        }
        stt<CPL>(tpw<Ty>(a.x_out) + o, xo);
        if constexpr (kDot) {
            if (a.dot) {
                const Vec<CPL> bb = ldt<CPL>(a.b + o);
#pragma unroll
                for (int i = 0; i < CPL; ++i) dotp[i] = add(dotp[i], mul(bb.v[i], xo.v[i]));
            }
        }
    } else {  // OP_CHEB_STEP  (solvers.py:559-571)
        const double dd = __ldg(a.d + row);
        Vec<CPL> r = ldt<CPL>(tp<Ty>(a.r_in) + o);
        Vec<CPL> dv = ldt<CPL>(tp<Ty>(a.xo) + o);
        Vec<CPL> xo = ldt_rw<CPL>(tp<Ty>(a.x_in) + o);
        Vec<CPL> dvn;
#pragma unroll
        for (int i = 0; i < CPL; ++i) {
            r.v[i] = sub(r.v[i], acc[i]);                                     // r -= A dv
            dvn.v[i] = add(mul(dv.v[i], a.c1), mul(a.c2, divd(r.v[i], dd)));  // dv*c1 + c2*(r/d)
            xo.v[i] = add(xo.v[i], dvn.v[i]);                                 // x += dv
        }
        stt<CPL>(tpw<Ty>(a.x_out) + o, xo);
        if (a.r_out) stt<CPL>(tpw<Ty>(a.r_out) + o, r);
        if (a.dv_out) stt<CPL>(tpw<Ty>(a.dv_out) + o, dvn);
        if constexpr (kDot) {
            if (a.dot) {
                Vec<CPL> bb = ldt<CPL>(a.b + o);
#pragma unroll
                for (int i = 0; i < CPL; ++i) dotp[i] = add(dotp[i], mul(bb.v[i], xo.v[i]));
            }
        }
    }
}

template <int OP, int CPL, typename Tx, typename Ty, class Src, int UNR = 4, int LM = 0>
__device__ __forceinline__ void do_row(const SpArgs& a, const Src& src, int row, int lo,
                                       int hi, int ld, int cofs, double (&dotp)[CPL]) {
    // 32-bit indices: rows, entries and element offsets < 2^31 (launch checks)
    const int o = row * ld + cofs;
    double acc[CPL];
    bool subtract;
    row_begin<OP, CPL, Ty>(a, o, acc, subtract);
    if constexpr (LM == 3) {
        if (subtract) row_accumulate_pairs<CPL, true, Tx, Src>(a, src, lo, hi, ld, cofs, acc);
        else row_accumulate_pairs<CPL, false, Tx, Src>(a, src, lo, hi, ld, cofs, acc);
    } else if (subtract)
        row_accumulate<CPL, true, Tx, Src, UNR, LM>(a, src, lo, hi, ld, cofs, acc);
    else
        row_accumulate<CPL, false, Tx, Src, UNR, LM>(a, src, lo, hi, ld, cofs, acc);
    row_end<OP, CPL, Tx, Ty>(a, row, o, acc, dotp);
}

// A long row (more than a.long_thr entries: AMG coarse operators carry rows
// of ~1000 entries among rows of ~60) by a whole CTA: all threads gather and
// multiply a chunk of the row's entries into shared memory (entry e, column
// c), then the row's LPR lane-threads fold the products in entry order --
// the same separately rounded mul then add/sub sequence as row_accumulate,
// so the result is bitwise that of the lane path, but the row's gathers run
// in parallel instead of as ceil(len/UNR) dependent rounds.
template <int M, int OP, typename Tv, typename Ti, typename Tx, typename Ty>
__device__ __forceinline__ void long_row_cta(const SpArgs& a, const GSrc<Tv, Ti>& src0, int row,
                                             double (&dotp)[Lay<M>::CPL]) {
    constexpr int CPL = Lay<M>::CPL, LPR = Lay<M>::LPR;
    constexpr int EPC = kLongProducts / M;          // entries per chunk
    // dynamic shared memory: launches without long rows reserve none, so the
    // lane path keeps its whole L1 for the gathered x rows
    extern __shared__ double s_p[];
    const int q = threadIdx.x;
    const GSrc<Tv, Ti> src = src0.at_row(a, row);
    const int lo = __ldg(a.rp + row), hi = __ldg(a.rp + row + 1);
    const int o = row * M + q * CPL;
    double acc[CPL];
    bool subtract = false;
    if (q < LPR) row_begin<OP, CPL, Ty>(a, o, acc, subtract);
    for (int k0 = lo; k0 < hi; k0 += EPC) {
        const int ne = min(EPC, hi - k0);
#pragma unroll 4
        for (int t = threadIdx.x; t < ne * M; t += kThreads) {
            const int e = t / M, c = t % M;
            s_p[t] = mul(src.val(k0 + e), (double)__ldg(tp<Tx>(a.x) + src.col(k0 + e) * M + c));
        }
        __syncthreads();
        if (q < LPR) {
            if (subtract) {
                for (int e = 0; e < ne; ++e)
#pragma unroll
                    for (int i = 0; i < CPL; ++i) acc[i] = sub(acc[i], s_p[e * M + q * CPL + i]);
            } else {
                for (int e = 0; e < ne; ++e)
#pragma unroll
                    for (int i = 0; i < CPL; ++i) acc[i] = add(acc[i], s_p[e * M + q * CPL + i]);
            }
        }
        __syncthreads();
    }
    if (q < LPR) row_end<OP, CPL, Tx, Ty>(a, row, o, acc, dotp);
}

// CTA-level fixed-shape reduction of the fused-dot partials (warp xor tree
// over row groups, then warps in order), finished by finish_reduction.
template <int M>
__device__ __forceinline__ void spmm_block_dot(const SpArgs& a, double (&dotp)[Lay<M>::CPL]) {
    constexpr int CPL = Lay<M>::CPL, LPR = Lay<M>::LPR;
    __shared__ double s_w[kThreads / 32][M];
    __shared__ double s_blk[M];
#pragma unroll
    for (int off = LPR; off < 32; off <<= 1)
#pragma unroll
        for (int i = 0; i < CPL; ++i)
            dotp[i] = add(dotp[i], __shfl_xor_sync(0xffffffffu, dotp[i], off));
    const int warp = threadIdx.x / 32, wl = threadIdx.x % 32;
    if (wl < LPR)
#pragma unroll
        for (int i = 0; i < CPL; ++i) s_w[warp][wl * CPL + i] = dotp[i];
    __syncthreads();
    if (threadIdx.x < M) {
        double acc = s_w[0][threadIdx.x];
        for (int w = 1; w < kThreads / 32; ++w) acc = add(acc, s_w[w][threadIdx.x]);
        s_blk[threadIdx.x] = acc;
    }
    __syncthreads();
    finish_reduction(a.red, s_blk, M, M);
}

// Occupancy floor per op: 6 CTAs/SM (<= 40 registers) for SpMV / Jacobi,
// 5 (<= 48) for the Chebyshev steps -- the largest that compile spill-free.
template <int M, int OP> constexpr int spmm_min_blocks() {
    if (M > 16) return 1;
    return (OP == OP_SPMV || OP == OP_JAC_SWEEP) ? 6 : 5;
}

// Operators with long rows on average (27-point stencils, the banded random
// C5 matrix: >= 12 entries per row): the LPR lanes of a row load LPR
// consecutive entries with ONE load each and exchange (column, value) by
// shuffles, instead of every lane loading every entry -- the replicated
// value loads were half of the kernel's L1 wavefronts (a warp's 8 rows sit
// in 8 different lines per entry).  Same entry order, same bits.  The trip
// count is warp-uniform (the warp's longest row); `live` rows accumulate.
template <int CPL, int LPR, class Src>
__device__ __forceinline__ void coop_accumulate(const SpArgs& a, const Src& src, int lo, int len,
                                                int ld, int cofs, bool live, bool subtract,
                                                double (&acc)[CPL]) {
    const int l = threadIdx.x % LPR;
    const int gbase = (threadIdx.x % 32) & ~(LPR - 1);
    const int wlen = __reduce_max_sync(0xffffffffu, len);
    for (int k = 0; k < wlen; k += LPR) {
        const int e = k + l;
        const int kk = e < len ? lo + e : lo;
        const int cm = len > 0 ? src.col(kk) : 0;
        const double vm = len > 0 ? src.val(kk) : 0.0;
        int c[LPR];
        double v[LPR];
#pragma unroll
        for (int u = 0; u < LPR; ++u) {
            c[u] = __shfl_sync(0xffffffffu, cm, gbase + u);
            v[u] = __shfl_sync(0xffffffffu, vm, gbase + u);
        }
        if (live && k < len) {
            Vec<CPL> g[LPR];
#pragma unroll
            for (int u = 0; u < LPR; ++u) g[u] = load_vec<CPL>(a.x + c[u] * ld + cofs);   // double only
            compiler_fence();
            if (subtract) {
#pragma unroll
                for (int u = 0; u < LPR; ++u)
                    if (k + u < len)
#pragma unroll
                        for (int i = 0; i < CPL; ++i) acc[i] = sub(acc[i], mul(v[u], g[u].v[i]));
            } else {
#pragma unroll
                for (int u = 0; u < LPR; ++u)
                    if (k + u < len)
#pragma unroll
                        for (int i = 0; i < CPL; ++i) acc[i] = add(acc[i], mul(v[u], g[u].v[i]));
            }
        }
    }
}

// LONG: small operators with long rows (AMG coarse levels, >= 12 nnz/row):
// 16 entries in flight per lane -- the row's dependent chain is 4x shorter;
// register-heavy, so only used where few CTAs run anyway.  Same order.
// COOP: large operators with long rows (coop_accumulate), M in {4, 8, 16}.
// COOP keeps the lane path's occupancy floor: at 4 CTAs/SM (no spills) the
// isolated product is faster, but whole C4 solves ran 2.8 % slower (A/B,
// profiles/r02_spmm_variants.txt).  Tx / Ty: vector types of
// the gathered operand / the row operands (double, or float levels of the
// fp32-vector V-cycle; COOP is double only).
template <int M, int OP, typename Tv, typename Ti, bool LONG = false, bool COOP = false,
          typename Tx = double, typename Ty = double, int LM = 0>
__global__ void __launch_bounds__(kThreads, LONG ? 1 : spmm_min_blocks<M, OP>())
spmm_kernel(SpArgs a) {
    pdl_enter();
    if (a.guard && *a.guard) return;
    using L = Lay<M>;
    constexpr int CPL = L::CPL, LPR = L::LPR, RPB = L::RPB;
    const int lane = threadIdx.x % LPR;
    const int cofs = lane * CPL;
    const GSrc<Tv, Ti> src{reinterpret_cast<const Ti*>(a.ci), reinterpret_cast<const Tv*>(a.vals)};
    double dotp[CPL];
#pragma unroll
    for (int i = 0; i < CPL; ++i) dotp[i] = 0.0;
    const int chunk = (int)a.chunk;
    const int rbeg = 0, rend = (int)a.nrows;
    const int gl = (int)gridDim.x - a.long_ctas;   // CTAs of the lane path
    if ((int)blockIdx.x >= gl) {
        // long rows: one CTA each (long_row_cta), strided over the long CTAs
        for (int j = (int)blockIdx.x - gl; j < a.n_long; j += a.long_ctas)
            long_row_cta<M, OP, Tv, Ti, Tx, Ty>(a, src, __ldg(a.long_rows + j), dotp);
    } else if constexpr (COOP) {
        const int lthr = a.n_long ? a.long_thr : 0x7fffffff;
        for (int r0 = rbeg + blockIdx.x * chunk; r0 < rend; r0 += gl * chunk) {
            const int r1 = min(r0 + chunk, rend);
            for (int rb = r0; rb < r1; rb += RPB) {            // warp-uniform passes
                const int row = rb + threadIdx.x / LPR;
                int lo = 0, len = 0;
                bool live = row < r1;
                if (live) {
                    lo = __ldg(a.rp + row);
                    len = __ldg(a.rp + row + 1) - lo;
                    if (len > lthr) { live = false; len = 0; }  // done by a long-row CTA
                }
                const GSrc<Tv, Ti> rs = live ? src.at_row(a, row) : src;
                const int o = row * M + cofs;
                double acc[CPL];
                bool subtract = false;
                if (live) row_begin<OP, CPL, double>(a, o, acc, subtract);
                coop_accumulate<CPL, LPR>(a, rs, lo, len, M, cofs, live, subtract, acc);
                if (live) row_end<OP, CPL, double, double>(a, row, o, acc, dotp);
            }
        }
    } else {
        const int lthr = a.n_long ? a.long_thr : 0x7fffffff;
        for (int r0 = rbeg + blockIdx.x * chunk; r0 < rend; r0 += gl * chunk) {
            const int r1 = min(r0 + chunk, rend);
            for (int row = r0 + threadIdx.x / LPR; row < r1; row += RPB) {
                const int lo = __ldg(a.rp + row), hi = __ldg(a.rp + row + 1);
                if (hi - lo > lthr) continue;            // done by a long-row CTA
                do_row<OP, CPL, Tx, Ty, GSrc<Tv, Ti>, LONG ? 16 : L::UNR, LM>(a, src.at_row(a, row), row, lo, hi,
                                                                  M, cofs, dotp);
            }
        }
    }
    if (a.dot) spmm_block_dot<M>(a, dotp);
}

// Generic m (any value, any layout): one thread per (row, column), thread
// t of a CTA owns column t % m for RPB = 256 / m rows.
template <int OP, typename Tv, typename Ti>
__global__ void __launch_bounds__(kThreads) spmm_kernel_generic(SpArgs a) {
    pdl_enter();
    if (a.guard && *a.guard) return;
    const int m = (int)a.m;
    const int rpb = kThreads / m;
    const int c = threadIdx.x % m;
    const GSrc<Tv, Ti> src{reinterpret_cast<const Ti*>(a.ci), reinterpret_cast<const Tv*>(a.vals)};
    double dotp[1] = {0.0};
    if (threadIdx.x < rpb * m) {
        const int chunk = (int)a.chunk;
        const int rbeg = 0, rend = (int)a.nrows;
        for (int r0 = rbeg + blockIdx.x * chunk; r0 < rend; r0 += gridDim.x * chunk) {
            const int r1 = min(r0 + chunk, rend);
            for (int row = r0 + threadIdx.x / m; row < r1; row += rpb) {
                do_row<OP, 1, double, double>(a, src.at_row(a, row), row, __ldg(a.rp + row),
                                              __ldg(a.rp + row + 1), m,
                              c, dotp);
            }
        }
    }
    {
        if (a.dot) {
            __shared__ double s_t[kThreads];
            __shared__ double s_blk[kMaxM];
            s_t[threadIdx.x] = dotp[0];
            __syncthreads();
            if (threadIdx.x < m) {
                double acc = s_t[threadIdx.x];
                for (int t = threadIdx.x + m; t < rpb * m; t += m) acc = add(acc, s_t[t]);
                s_blk[threadIdx.x] = acc;
            }
            __syncthreads();
            finish_reduction(a.red, s_blk, m, m);
        }
    }
}


}  // namespace mrs
