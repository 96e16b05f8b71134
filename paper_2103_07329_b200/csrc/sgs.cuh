// sgs.cuh -- Gauss-Seidel half-sweeps in the reference's exact sequential
// row order (blas2.sgs_sweep, src/blas2.py:113-162, kernel gs_sweep,
// _ckernels.pyx:60-79), parallelised by level scheduling.
//
// With the reference's default one-leaf topology the hybrid Gauss-Seidel
// sweep is plain sequential Gauss-Seidel over the whole level.  Row i reads
// the NEW value of every column it references that the sequential order
// visits before i and the OLD value of every column visited after i.  The
// host (solver.cu, build_sgs_schedule) assigns each row the smallest level
// greater than the levels of both kinds of neighbours visited before it
// (true dependences AND rows that must still see its old value), so rows of
// one level touch no common unknowns and every row reads exactly the values
// the sequential sweep would: bitwise the reference.
//
// One launch per half-sweep on ONE thread-block cluster: the cluster's CTAs
// split each level's rows and meet at a cluster barrier between levels (the
// barrier's acquire side makes other CTAs' writes visible to plain loads;
// see tail.cuh).  Per row: v = b - 0 (the off-leaf coupling of one leaf is
// zero), v -= a_ik x_k in entry order skipping the diagonal, x_i = v / a_ii.
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
    const int32_t* order;       // rows grouped by level, ascending inside a level
    const int32_t* lptr;        // [nlev + 1] level boundaries in `order`
    int nlev;
    const int32_t* dpos;        // absolute entry index of each row's diagonal
    const double* d;            // diagonal values (stored value widened)
    const double* b;
    const double* c;            // off-leaf coupling (plugin gs_sweep); null = 0
    double* x;
    int m;
    int nrows;
    const int* guard;
};

template <int CPL, typename Tv, typename Ti>
__device__ __forceinline__ void sgs_row(const SgsArgs& a, int row, int cofs) {
    const Ti* __restrict__ ci = reinterpret_cast<const Ti*>(a.ci);
    const Tv* __restrict__ vv = reinterpret_cast<const Tv*>(a.vals);
    const int m = a.m;
    const int lo = __ldg(a.rp + row), hi = __ldg(a.rp + row + 1), dp = __ldg(a.dpos + row);
    const int base = a.slab_base ? __ldg(a.slab_base + (row >> a.slab_shift)) : 0;
    Vec<CPL> v = load_vec<CPL>(a.b + (int64_t)row * m + cofs);
    if (a.c) {                                                     // v = b - c
        const Vec<CPL> cc = load_vec<CPL>(a.c + (int64_t)row * m + cofs);
#pragma unroll
        for (int i = 0; i < CPL; ++i) v.v[i] = sub(v.v[i], cc.v[i]);
    }                                                              // (b - 0.0 == b)
    for (int k = lo; k < hi; k += 4) {
        int c[4];
        double w[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int kk = (k + u < hi) ? k + u : lo;
            c[u] = base + (int)__ldg(ci + kk);
            w[u] = widen(__ldg(vv + kk));
        }
        compiler_fence();
        Vec<CPL> g[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) g[u] = load_vec_rw<CPL>(a.x + (int64_t)c[u] * m + cofs);
        compiler_fence();
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (k + u < hi && k + u != dp) {
#pragma unroll
                for (int i = 0; i < CPL; ++i) v.v[i] = sub(v.v[i], mul(w[u], g[u].v[i]));
            }
        }
    }
    const double dd = __ldg(a.d + row);
#pragma unroll
    for (int i = 0; i < CPL; ++i) v.v[i] = divd(v.v[i], dd);
    store_vec<CPL>(a.x + (int64_t)row * m + cofs, v);
}

// CPL columns per lane (2 when m is even), m / CPL lanes per row.
template <int CPL, typename Tv, typename Ti>
__global__ void __launch_bounds__(kThreads) sgs_kernel(SgsArgs a) {
    if (a.guard && *a.guard) return;     // same value in every CTA: all skip together
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    const int crank = (int)cl.block_rank(), csize = (int)cl.num_blocks();
    const int lpr = a.m / CPL, rpb = kThreads / lpr;
    const int rs = threadIdx.x / lpr, cofs = (threadIdx.x % lpr) * CPL;
    for (int lev = 0; lev < a.nlev; ++lev) {
        const int lo = __ldg(a.lptr + lev), hi = __ldg(a.lptr + lev + 1);
        if (rs < rpb)
            for (int idx = lo + crank * rpb + rs; idx < hi; idx += csize * rpb)
                sgs_row<CPL, Tv, Ti>(a, __ldg(a.order + idx), cofs);
        cl.sync();
    }
}

// Small or narrow levels (few rows per schedule level, e.g. AMG coarse
// levels): ONE CTA of kSgsCta threads walks all schedule levels with
// __syncthreads between them -- a block barrier instead of a cluster
// barrier, and the level's vectors stay in this SM's L1 (coherent for the
// block's own writes).
constexpr int kSgsCta = 1024;

template <int CPL, typename Tv, typename Ti>
__global__ void __launch_bounds__(kSgsCta) sgs_cta_kernel(SgsArgs a) {
    if (a.guard && *a.guard) return;
    const int lpr = a.m / CPL, rpb = kSgsCta / lpr;
    const int rs = threadIdx.x / lpr, cofs = (threadIdx.x % lpr) * CPL;
    for (int lev = 0; lev < a.nlev; ++lev) {
        const int lo = __ldg(a.lptr + lev), hi = __ldg(a.lptr + lev + 1);
        if (rs < rpb)
            for (int idx = lo + rs; idx < hi; idx += rpb)
                sgs_row<CPL, Tv, Ti>(a, __ldg(a.order + idx), cofs);
        __syncthreads();
    }
}

}  // namespace mrs
