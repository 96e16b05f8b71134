// sgs.cuh -- Gauss-Seidel half-sweeps in the reference's exact sequential
// row order (blas2.sgs_sweep, src/blas2.py:113-162, kernel gs_sweep,
// _ckernels.pyx:60-79), parallelised by level scheduling.
//
// With the reference's default one-leaf topology the hybrid Gauss-Seidel
// sweep is plain sequential Gauss-Seidel over the whole level.  Row i reads
// the NEW value of every column it references that the sequential order
// visits before i and the OLD value of every column visited after i.  The
// host (sgs_sched.h) assigns each row the smallest schedule level greater
// than the levels of both kinds of neighbours visited before it (true
// dependences AND rows that must still see its old value), so rows of one
// level touch no common unknowns and every row reads exactly the values the
// sequential sweep would: bitwise the reference.
//
// Per row: v = b - c (c = the off-leaf coupling: zero for one leaf, and
// b - 0.0 == b), v -= a_ik x_k in entry order skipping the diagonal,
// x_i = v / a_ii.
//
// Latency: a schedule level is one dependent step, so the walk is a
// software pipeline across levels -- the row descriptor (row, extent,
// diagonal; int4, schedule order) of level L+2 and everything of level L+1
// that does not depend on x (b - c, the first kPre (column, value) entries)
// are loaded while level L is computed; after each barrier only the x
// gathers of the row remain on the critical path.
#pragma once

#include <cooperative_groups.h>

#include "spmm.cuh"

namespace mrs {

struct SgsArgs {
    const int32_t* rp;
    const void* ci;
    const void* vals;
    const int32_t* slab_base;   // slab-relative 16-bit columns (optional)
    int slab_shift;
    const int4* meta;           // schedule order: (row, first entry, end entry, diagonal entry)
    const int32_t* lptr;        // [nlev + 1] level boundaries in `meta`
    int nlev;
    const double* d;            // diagonal values (stored value widened)
    const double* b;
    const double* c;            // off-leaf coupling (plugin gs_sweep); null = 0
    double* x;
    int m;
    int nrows;
    const int* guard;
};

constexpr int kPre = 8;        // entries of a row fetched ahead of its level

template <int CPL> struct SgsPre {
    int4 md;                    // row, lo, hi, dp
    Vec<CPL> v;                 // b - c
    uint32_t craw[kPre];        // raw column indices (slab base added at use)
    double w[kPre];
    int base;
    bool ok;
};

template <typename Ti>
__device__ __forceinline__ uint32_t ld_idx(const void* ci, int k) {
    return (uint32_t)__ldg(reinterpret_cast<const Ti*>(ci) + k);
}
template <typename Tv>
__device__ __forceinline__ double ld_val(const void* v, int k) {
    return widen(__ldg(reinterpret_cast<const Tv*>(v) + k));
}

// Loads of a row that do not depend on x.
template <int CPL, typename Tv, typename Ti>
__device__ __forceinline__ void sgs_fetch(const SgsArgs& a, const int4 md, bool ok, int cofs,
                                          SgsPre<CPL>& p) {
    p.ok = ok;
    p.md = md;
    if (!ok) return;
    const int row = md.x, lo = md.y, hi = md.z;
    p.base = a.slab_base ? __ldg(a.slab_base + (row >> a.slab_shift)) : 0;
    p.v = load_vec<CPL>(a.b + (int64_t)row * a.m + cofs);
    if (a.c) {
        const Vec<CPL> cc = load_vec<CPL>(a.c + (int64_t)row * a.m + cofs);
#pragma unroll
        for (int i = 0; i < CPL; ++i) p.v.v[i] = sub(p.v.v[i], cc.v[i]);
    }
#pragma unroll
    for (int u = 0; u < kPre; ++u) {
        const int kk = (lo + u < hi) ? lo + u : lo;
        p.craw[u] = ld_idx<Ti>(a.ci, kk);
        p.w[u] = ld_val<Tv>(a.vals, kk);
    }
}

// Accumulate and store a fetched row: the kPre gathers at once, the rest of a
// long row in groups of 8 (entry order throughout), x_i = v / a_ii.
template <int CPL, typename Tv, typename Ti>
__device__ __forceinline__ void sgs_finish(const SgsArgs& a, SgsPre<CPL>& p, int cofs) {
    const int m = a.m;
    const int row = p.md.x, lo = p.md.y, hi = p.md.z, dp = p.md.w;
    Vec<CPL> g[kPre];
#pragma unroll
    for (int u = 0; u < kPre; ++u)
        g[u] = load_vec_rw<CPL>(a.x + (int64_t)(p.base + (int)p.craw[u]) * m + cofs);
    compiler_fence();
#pragma unroll
    for (int u = 0; u < kPre; ++u)
        if (lo + u < hi && lo + u != dp)
#pragma unroll
            for (int i = 0; i < CPL; ++i) p.v.v[i] = sub(p.v.v[i], mul(p.w[u], g[u].v[i]));
    for (int k = lo + kPre; k < hi; k += 8) {
        int c[8];
        double w[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int kk = (k + u < hi) ? k + u : lo;
            c[u] = p.base + (int)ld_idx<Ti>(a.ci, kk);
            w[u] = ld_val<Tv>(a.vals, kk);
        }
        compiler_fence();
        Vec<CPL> h[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) h[u] = load_vec_rw<CPL>(a.x + (int64_t)c[u] * m + cofs);
        compiler_fence();
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (k + u < hi && k + u != dp)
#pragma unroll
                for (int i = 0; i < CPL; ++i) p.v.v[i] = sub(p.v.v[i], mul(w[u], h[u].v[i]));
    }
    const double dd = __ldg(a.d + row);
#pragma unroll
    for (int i = 0; i < CPL; ++i) p.v.v[i] = divd(p.v.v[i], dd);
    store_vec<CPL>(a.x + (int64_t)row * m + cofs, p.v);
}

// Row descriptor `first` of level `lev` (ok = the level has that many rows).
__device__ __forceinline__ int4 sgs_meta(const SgsArgs& a, int lev, int first, bool& ok) {
    ok = false;
    if (lev >= a.nlev) return make_int4(0, 0, 0, 0);
    const int idx = __ldg(a.lptr + lev) + first;
    ok = idx < __ldg(a.lptr + lev + 1);
    return ok ? __ldg(a.meta + idx) : make_int4(0, 0, 0, 0);
}

// The schedule walk shared by both launch shapes: this thread's rows of a
// level are entries first, first + stride, ... of the level's meta range.
template <int CPL, typename Tv, typename Ti, class Barrier>
__device__ __forceinline__ void sgs_walk(const SgsArgs& a, int first, int stride, int cofs,
                                         bool active, Barrier barrier) {
    SgsPre<CPL> cur, nxt;
    bool ok0 = false, ok1 = false, ok2 = false;
    int4 m1 = make_int4(0, 0, 0, 0);
    cur.ok = false;
    if (active) {
        const int4 m0 = sgs_meta(a, 0, first, ok0);
        m1 = sgs_meta(a, 1, first, ok1);
        sgs_fetch<CPL, Tv, Ti>(a, m0, ok0, cofs, cur);
    }
    for (int lev = 0; lev < a.nlev; ++lev) {
        if (active) {
            // in flight while this level computes: data of lev+1, descriptor of lev+2
            sgs_fetch<CPL, Tv, Ti>(a, m1, ok1, cofs, nxt);
            const int4 m2 = sgs_meta(a, lev + 2, first, ok2);
            compiler_fence();
            if (cur.ok) sgs_finish<CPL, Tv, Ti>(a, cur, cofs);
            // further rows of this thread in a wide level (no lookahead)
            const int hi = __ldg(a.lptr + lev + 1);
            for (int idx = __ldg(a.lptr + lev) + first + stride; idx < hi; idx += stride) {
                SgsPre<CPL> q;
                sgs_fetch<CPL, Tv, Ti>(a, __ldg(a.meta + idx), true, cofs, q);
                sgs_finish<CPL, Tv, Ti>(a, q, cofs);
            }
            cur = nxt;
            m1 = m2;
            ok1 = ok2;
        }
        barrier();
    }
}

// CPL columns per lane (2 when m is even), m / CPL lanes per row.  One
// thread-block cluster; cluster barrier between schedule levels (its acquire
// side -- MEMBAR.GPU + CCTL.IVALL (L1 invalidate) in SASS -- makes other
// CTAs' writes visible to plain loads).
template <int CPL, typename Tv, typename Ti>
__global__ void __launch_bounds__(kThreads) sgs_kernel(SgsArgs a) {
    if (a.guard && *a.guard) return;     // same value in every CTA: all skip together
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    const int crank = (int)cl.block_rank(), csize = (int)cl.num_blocks();
    const int lpr = a.m / CPL, rpb = kThreads / lpr;
    const int rs = threadIdx.x / lpr, cofs = (threadIdx.x % lpr) * CPL;
    sgs_walk<CPL, Tv, Ti>(a, crank * rpb + rs, csize * rpb, cofs, rs < rpb, [&]() { cl.sync(); });
}

// Narrow levels (few rows per schedule level, e.g. AMG coarse levels): ONE
// CTA walks all schedule levels with __syncthreads between them -- a block
// barrier instead of a cluster barrier, and the level's vectors stay in this
// SM's L1 (coherent for the block's own writes).
constexpr int kSgsCta = 512;

template <int CPL, typename Tv, typename Ti>
__global__ void __launch_bounds__(kSgsCta) sgs_cta_kernel(SgsArgs a) {
    if (a.guard && *a.guard) return;
    const int lpr = a.m / CPL, rpb = kSgsCta / lpr;
    const int rs = threadIdx.x / lpr, cofs = (threadIdx.x % lpr) * CPL;
    sgs_walk<CPL, Tv, Ti>(a, rs, rpb, cofs, rs < rpb, []() { __syncthreads(); });
}

}  // namespace mrs
