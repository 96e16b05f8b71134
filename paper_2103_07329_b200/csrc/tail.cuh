// tail.cuh -- the coarse end of the V-cycle in ONE launch.
//
// Levels with few rows (<= tail_rows) are latency-bound: each of their ~10
// kernels per V-cycle costs a launch and a drain for a few thousand rows.
// The tail kernel runs the whole sub-V-cycle below a level (pre-smoothing,
// residual, restriction, coarse solve, prolongation, post-smoothing -- the
// same steps, same arithmetic, recorded from the schedule builder) on one
// thread-block CLUSTER: the cluster's CTAs split each step's rows and meet at
// a hardware cluster barrier (barrier.cluster arrive.release / wait.acquire)
// between steps.  The barrier's acquire invalidates L1 (CCTL.IVALL in SASS),
// so plain loads see what other CTAs of the cluster wrote in earlier steps.
#pragma once

#include <cooperative_groups.h>

#include "spmm.cuh"

namespace mrs {

enum TailKind : int { TK_SPMM = 0, TK_COARSE = 1 };

struct TailStep {
    int kind;
    int op;            // SpOp (TK_SPMM)
    int vb, ib;        // matrix value / index bytes
    SpArgs a;          // matrix arrays + operands
    const double* inv; // TK_COARSE: x = inv b (nc x nc)
    int64_t nc;
    const double* cb;
    double* cx;
};

template <int M, int OP, typename Tv, typename Ti>
__device__ __forceinline__ void tail_rows(const SpArgs& a, int crank, int csize) {
    using L = Lay<M>;
    constexpr int CPL = L::CPL, LPR = L::LPR, RPB = L::RPB;
    const int cofs = (threadIdx.x % LPR) * CPL;
    const GSrc<Tv, Ti> src{reinterpret_cast<const Ti*>(a.ci), reinterpret_cast<const Tv*>(a.vals)};
    double dotp[CPL];
    for (int row = crank * RPB + threadIdx.x / LPR; row < (int)a.nrows; row += csize * RPB)
        do_row<OP, CPL, GSrc<Tv, Ti>, 4, false>(a, src.at_row(a, row), row, __ldg(a.rp + row),
                                                __ldg(a.rp + row + 1), M, cofs, dotp);
}

template <int M, int OP>
__device__ __forceinline__ void tail_dispatch_t(const TailStep& st, int crank, int csize) {
    if (st.vb == 8) {
        if (st.ib == 2) tail_rows<M, OP, double, uint16_t>(st.a, crank, csize);
        else tail_rows<M, OP, double, uint32_t>(st.a, crank, csize);
    } else {
        if (st.ib == 2) tail_rows<M, OP, float, uint16_t>(st.a, crank, csize);
        else tail_rows<M, OP, float, uint32_t>(st.a, crank, csize);
    }
}

// x = inv b: rows i = crank, crank + csize, ...; thread (ks, c) folds k for
// column c, partials folded in order (same shape as coarse_kernel).
__device__ __forceinline__ void tail_coarse(const TailStep& st, int m, int crank, int csize) {
    __shared__ double s_t[kThreads];
    const int kpb = kThreads / m;
    const int c = threadIdx.x % m, ks = threadIdx.x / m;
    for (int64_t i = crank; i < st.nc; i += csize) {
        double acc = 0.0;
        if (ks < kpb)
            for (int64_t k = ks; k < st.nc; k += kpb)
                acc = add(acc, mul(__ldg(st.inv + i * st.nc + k), st.cb[k * m + c]));
        s_t[threadIdx.x] = acc;
        __syncthreads();
        if (threadIdx.x < m) {
            double t = s_t[threadIdx.x];
            for (int q = 1; q < kpb; ++q) t = add(t, s_t[q * m + threadIdx.x]);
            st.cx[i * m + threadIdx.x] = t;
        }
        __syncthreads();
    }
}

template <int M>
__global__ void __launch_bounds__(kThreads) tail_kernel(const TailStep* __restrict__ steps,
                                                        int nsteps, const int* guard) {
    if (guard && *guard) return;     // same value in every CTA: all skip together
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    const int crank = (int)cl.block_rank(), csize = (int)cl.num_blocks();
    for (int s = 0; s < nsteps; ++s) {
        const TailStep& st = steps[s];
        if (st.kind == TK_COARSE) {
            tail_coarse(st, M, crank, csize);
        } else {
            switch (st.op) {
            case OP_SPMV: tail_dispatch_t<M, OP_SPMV>(st, crank, csize); break;
            case OP_JAC_SWEEP: tail_dispatch_t<M, OP_JAC_SWEEP>(st, crank, csize); break;
            case OP_CHEB_FIRST: tail_dispatch_t<M, OP_CHEB_FIRST>(st, crank, csize); break;
            case OP_CHEB_STEP: tail_dispatch_t<M, OP_CHEB_STEP>(st, crank, csize); break;
            }
        }
        cl.sync();
    }
}

}  // namespace mrs
