// reduce.cuh -- deterministic multi-column reductions with a fused scalar
// epilogue, and the per-solve device state the epilogues update.
//
// Every reduction in the solve path (dot, norm2, dot_many of the reference,
// src/blas.py:173-221) is finished on the device in one kernel:
//   thread partials -> warp/block tree (fixed shape) -> per-CTA partial row
//   -> the last CTA to arrive (atomic ticket) folds the CTA partials in CTA
//   order and runs the scalar epilogue (the reference's _coef / convergence
//   test, src/solvers.py:111-123, :171, :180) on the reduced values.
// Results depend only on (n, m, grid), never on scheduling: deterministic.
#pragma once

#include "common.cuh"

namespace mrs {

// Per-solve scalar state (device memory).  m <= kMaxM columns.
constexpr int kMaxM = 64;

struct SolveState {
    double bscale[kMaxM];    // ||b_j|| or 1 (solvers._b_scale)
    double rnorm[kMaxM];
    double rho[kMaxM];
    double rho_next[kMaxM];
    double alpha[kMaxM];
    double neg_alpha[kMaxM];
    double beta[kMaxM];
    double omega[kMaxM];
    double neg_omega[kMaxM];
    double final_rel[kMaxM];
    double tol;
    int m;
    int max_iters;
    int it;                  // completed-iteration counter (reference `it`)
    int skip;                // remaining kernels of this iteration are no-ops
    int stop;                // loop ends after this iteration
    int err;                 // MRS_OK / MRS_ERR_BREAKDOWN
    int err_col;
    int err_site;
    int merged;              // BiCGStab merged variant (snorm always from (s,s))
    int pskip;               // RBiCGStab: skip the end-of-iteration p update
    int nodrift;             // PBiCGStab: skip this iteration's drift check
    double drift_limit;      // PBiCGStab DRIFT_LIMIT (solvers.py:68)
    double one[kMaxM];       // per-column constants for axpby-shaped steps
    double neg_one[kMaxM];
    int has_cond;            // graph conditional handle valid
    cudaGraphConditionalHandle cond;
    double* history;         // (max_iters + 1) * m, device
};

enum Epilogue : int {
    EPI_NONE = 0,
    EPI_BSCALE,        // out = b.b            -> bscale
    EPI_RNORM_INIT,    // out = r.r            -> rnorm, history[0], stop
    EPI_RHO,           // out = r.z            -> rho
    EPI_CG_ALPHA,      // out = p.q            -> it++, alpha = rho / pq
    EPI_CG_RNORM,      // out = r.r            -> rnorm, history[it], skip/stop
    EPI_CG_BETA,       // out = r.z            -> beta = rho_new / rho, rho = rho_new
    EPI_BICG_ALPHA,    // out = r0.v           -> it++, alpha = rho / rv
    EPI_BICG_OMEGA,    // out = (t.s, t.t, s.s) -> omega
    EPI_BICG_RNORM,    // out = (r0.r, r.r)   -> rnorm, history, stop, beta
    EPI_FINAL,         // out = r.r (true residual) -> final_rel
    EPI_CG_RNORM_BETA, // out = (r.r, r.z)     -> EPI_CG_RNORM then, if not converged, EPI_CG_BETA
    EPI_CG_RNORM_BETA1,// out = r.r, z = r (no preconditioner): same with r.z = r.r
    // reordered BiCGStab (solvers.py:296-364)
    EPI_RBICG_OMEGA,   // out = (t.s, t.t, r0.s, r0.t, s.s) -> omega, rho', rnorm, history,
                       //   stop; beta, rho while not converged
    // pipelined BiCGStab (solvers.py:367-479)
    EPI_PBICG_INIT,    // out = (r0.r, r0.w)  -> rho, alpha
    EPI_PBICG_OMEGA,   // out = (q.y, y.y)    -> it++, omega
    EPI_PBICG_RHO,     // out = (r0.r, r0.w, r0.s, r0.z, r.r) -> rnorm, history, beta,
                       //   alpha, rho, stop, drift-check flag
    EPI_PBICG_DRIFT,   // out = chk.chk       -> instability check
    EPI_STAT_RNORM,    // out = r.r (true residual) -> it++, rnorm, history, stop
};
constexpr int kMaxK = 5;   // reduced values per column of one reduction

// Breakdown sites, reported to the host for the exception message.
enum BreakSite : int {
    BRK_CG_CURVATURE = 1, BRK_CG_RHO = 2, BRK_BICG_RV = 3, BRK_BICG_OMEGA = 4,
    BRK_BICG_RHO = 5, BRK_BICG_OMEGA_PREV = 6, BRK_PBICG_R0W = 7, BRK_PBICG_R0S = 8,
};

struct RedArgs {
    double* partials;        // [gridDim.x][K * m]
    unsigned int* ticket;    // zero between uses; reset by the last CTA
    double* out;             // [K * m] reduced values (device)
    SolveState* st;          // may be null for EPI_NONE
    int epi;
};

// _coef (solvers.py:111-123): num/den, zero den with nonzero rnorm is a
// breakdown, zero den on a converged column yields 0.
static __device__ __forceinline__ double coef(double num, double den, double rnorm, int c,
                                       SolveState* st, int site, bool& bad) {
    if (den == 0.0) {
        if (rnorm > 0.0) {
            bad = true;
            atomicMin(&st->err_col, c);
            st->err_site = site;
        }
        return 0.0;
    }
    return divd(num, den);
}

static __device__ __forceinline__ void set_loop(SolveState* st, bool keep_going) {
    if (st->has_cond) cudaGraphSetConditional(st->cond, keep_going ? 1u : 0u);
}

// Runs on ONE block (the last to arrive), all threads; `v` = reduced values
// in shared memory, laid out [K][m].
static __device__ void run_epilogue(int epi, SolveState* st, const double* v, int m) {
    const int c = threadIdx.x;
    const bool act = c < m;
    bool bad = false;
    switch (epi) {
    case EPI_NONE:
        break;
    case EPI_BSCALE:
        if (act) { double nb = sqrt(v[c]); st->bscale[c] = nb > 0.0 ? nb : 1.0; }
        break;
    case EPI_RNORM_INIT: {
        bool conv = true;
        if (act) {
            double rn = sqrt(v[c]);
            st->rnorm[c] = rn;
            st->history[c] = divd(rn, st->bscale[c]);
            conv = rn <= mul(st->tol, st->bscale[c]);
        }
        int all = __syncthreads_and(conv);
        if (threadIdx.x == 0) {
            st->it = 0; st->skip = 0; st->err = MRS_OK; st->err_col = 1 << 30; st->err_site = 0;
            st->pskip = 0; st->nodrift = 1;
            st->stop = (all || st->max_iters <= 0) ? 1 : 0;
            set_loop(st, !st->stop);
        }
        return;
    }
    case EPI_RHO:
        if (act) st->rho[c] = v[c];
        break;
    case EPI_CG_ALPHA:
        if (act) {
            double a = coef(st->rho[c], v[c], st->rnorm[c], c, st, BRK_CG_CURVATURE, bad);
            st->alpha[c] = a; st->neg_alpha[c] = -a;
        }
        if (threadIdx.x == 0) st->it += 1;
        break;
    case EPI_STAT_RNORM:
    case EPI_CG_RNORM: {
        bool conv = true;
        if (epi == EPI_STAT_RNORM) {
            if (threadIdx.x == 0) st->it += 1;
            __syncthreads();
        }
        if (act) {
            double rn = sqrt(v[c]);
            st->rnorm[c] = rn;
            st->history[(size_t)st->it * m + c] = divd(rn, st->bscale[c]);
            conv = rn <= mul(st->tol, st->bscale[c]);
        }
        int all = __syncthreads_and(conv);
        if (threadIdx.x == 0) {
            if (all) { st->skip = 1; st->stop = 1; }
            else if (st->it >= st->max_iters) st->stop = 1;
            set_loop(st, !st->stop);
        }
        return;
    }
    case EPI_CG_RNORM_BETA:
    case EPI_CG_RNORM_BETA1: {
        const int zo = epi == EPI_CG_RNORM_BETA ? m : 0;
        bool conv = true;
        if (act) {
            double rn = sqrt(v[c]);
            st->rnorm[c] = rn;
            st->history[(size_t)st->it * m + c] = divd(rn, st->bscale[c]);
            conv = rn <= mul(st->tol, st->bscale[c]);
        }
        int all = __syncthreads_and(conv);
        if (!all && act) {
            st->beta[c] = coef(v[zo + c], st->rho[c], st->rnorm[c], c, st, BRK_CG_RHO, bad);
            st->rho[c] = v[zo + c];
        }
        int anybad = __syncthreads_or(bad);
        if (threadIdx.x == 0) {
            if (all) { st->skip = 1; st->stop = 1; }
            else if (st->it >= st->max_iters) st->stop = 1;
            if (anybad) { st->err = MRS_ERR_BREAKDOWN; st->skip = 1; st->stop = 1; }
            set_loop(st, !st->stop);
        }
        return;
    }
    case EPI_CG_BETA:
        if (act) {
            st->beta[c] = coef(v[c], st->rho[c], st->rnorm[c], c, st, BRK_CG_RHO, bad);
            st->rho[c] = v[c];
        }
        break;
    case EPI_BICG_ALPHA:
        if (act) {
            double a = coef(st->rho[c], v[c], st->rnorm[c], c, st, BRK_BICG_RV, bad);
            st->alpha[c] = a; st->neg_alpha[c] = -a;
        }
        if (threadIdx.x == 0) st->it += 1;
        break;
    case EPI_BICG_OMEGA: {
        // solvers.py:271-275: ||s|| replaces rnorm in the breakdown test
        // only when np.any(tt == 0) over all columns.
        int anyz = __syncthreads_or(act && v[m + c] == 0.0);
        if (act) {
            double ts = v[c], tt = v[m + c], ss = v[2 * m + c];
            double snorm = (anyz || st->merged) ? sqrt(ss) : st->rnorm[c];
            double w = coef(ts, tt, snorm, c, st, BRK_BICG_OMEGA, bad);
            st->omega[c] = w; st->neg_omega[c] = -w;
        }
        break;
    }
    case EPI_BICG_RNORM: {
        bool conv = true;
        if (act) {
            double rr = v[m + c];
            double rn = sqrt(rr > 0.0 ? rr : 0.0);
            st->rnorm[c] = rn;
            st->rho_next[c] = v[c];
            st->history[(size_t)st->it * m + c] = divd(rn, st->bscale[c]);
            conv = rn <= mul(st->tol, st->bscale[c]);
        }
        int all = __syncthreads_and(conv);
        int cont = !all && (st->it < st->max_iters);
        if (cont && act) {
            // next iteration's beta (solvers.py:246-249), evaluated only when
            // the loop continues, exactly like the reference.
            double rp = st->rho[c];
            double rn_ = st->rho_next[c];
            double b1 = coef(rn_, rp, st->rnorm[c], c, st, BRK_BICG_RHO, bad);
            double b2 = coef(st->alpha[c], st->omega[c], st->rnorm[c], c, st,
                             BRK_BICG_OMEGA_PREV, bad);
            st->beta[c] = mul(b1, b2);
            st->rho[c] = rn_;
        }
        int anybad = __syncthreads_or(bad);
        if (threadIdx.x == 0) {
            st->stop = cont ? 0 : 1;
            if (anybad) { st->err = MRS_ERR_BREAKDOWN; st->stop = 1; st->skip = 1; }
            set_loop(st, !st->stop);
        }
        return;
    }
    case EPI_FINAL:
        if (act) st->final_rel[c] = divd(sqrt(v[c]), st->bscale[c]);
        break;
    case EPI_RBICG_OMEGA: {
        // solvers.py:334-359.  omega breaks down BEFORE the X/r update (skip
        // everything); beta after it (the update still runs, p does not).
        double w = 0.0, rn = 0.0;
        if (act) {
            const double ts = v[c], tt = v[m + c], r0s = v[2 * m + c], r0t = v[3 * m + c];
            const double ss = v[4 * m + c];
            w = coef(ts, tt, sqrt(ss), c, st, BRK_BICG_OMEGA, bad);
            st->omega[c] = w; st->neg_omega[c] = -w;
            st->rho_next[c] = sub(r0s, mul(w, r0t));
            // max(ss - 2 omega ts + omega^2 tt, 0), numpy's left-to-right order
            double rr = add(sub(ss, mul(mul(2.0, w), ts)), mul(mul(w, w), tt));
            rr = (rr != rr) ? rr : (rr > 0.0 ? rr : 0.0);
            rn = sqrt(rr);
        }
        if (__syncthreads_or(bad)) break;          // omega breakdown: common path below
        bool conv = true;
        if (act) {
            st->rnorm[c] = rn;
            st->history[(size_t)st->it * m + c] = divd(rn, st->bscale[c]);
            conv = rn <= mul(st->tol, st->bscale[c]);
        }
        const int all = __syncthreads_and(conv);
        if (!all) {
            // beta = coef(rho', rho) * coef(alpha, omega); the first factor's
            // breakdown is reported before the second's (like the reference)
            double b1 = 0.0;
            if (act) b1 = coef(st->rho_next[c], st->rho[c], rn, c, st, BRK_BICG_RHO, bad);
            if (!__syncthreads_or(bad) && act) {
                const double b2 = coef(st->alpha[c], w, rn, c, st, BRK_BICG_OMEGA_PREV, bad);
                st->beta[c] = mul(b1, b2);
                st->rho[c] = st->rho_next[c];
            }
        }
        const int anybad = __syncthreads_or(bad);
        if (threadIdx.x == 0) {
            st->pskip = (all || anybad) ? 1 : 0;
            st->stop = (all || anybad || st->it >= st->max_iters) ? 1 : 0;
            if (anybad) st->err = MRS_ERR_BREAKDOWN;
            set_loop(st, !st->stop);
        }
        return;
    }
    case EPI_PBICG_INIT:
        // solvers.py:401-402
        if (act) {
            st->rho[c] = v[c];
            const double a = coef(v[c], v[m + c], st->rnorm[c], c, st, BRK_PBICG_R0W, bad);
            st->alpha[c] = a; st->neg_alpha[c] = -a;
            st->omega[c] = 0.0; st->neg_omega[c] = -0.0;
        }
        if (threadIdx.x == 0) st->nodrift = 1;
        break;
    case EPI_PBICG_OMEGA:
        // solvers.py:443-445
        if (act) {
            const double w = coef(v[c], v[m + c], st->rnorm[c], c, st, BRK_BICG_OMEGA, bad);
            st->omega[c] = w; st->neg_omega[c] = -w;
        }
        if (threadIdx.x == 0) st->it += 1;
        break;
    case EPI_PBICG_RHO: {
        // solvers.py:461-472 (evaluated every iteration, converged or not)
        bool conv = true;
        double rn = 0.0;
        if (act) {
            const double rr = v[4 * m + c];
            rn = sqrt((rr != rr) ? rr : (rr > 0.0 ? rr : 0.0));
            st->rnorm[c] = rn;
            st->history[(size_t)st->it * m + c] = divd(rn, st->bscale[c]);
            conv = rn <= mul(st->tol, st->bscale[c]);
        }
        const int all = __syncthreads_and(conv);
        double b1 = 0.0, beta = 0.0;
        if (act) b1 = coef(v[c], st->rho[c], rn, c, st, BRK_BICG_RHO, bad);
        if (!__syncthreads_or(bad)) {
            if (act) beta = mul(b1, coef(st->alpha[c], st->omega[c], rn, c, st,
                                         BRK_BICG_OMEGA_PREV, bad));
            if (!__syncthreads_or(bad) && act) {
                const double r0w = v[m + c], r0s = v[2 * m + c], r0z = v[3 * m + c];
                const double r0s_next = add(r0w, mul(beta, sub(r0s, mul(st->omega[c], r0z))));
                const double a = coef(v[c], r0s_next, rn, c, st, BRK_PBICG_R0S, bad);
                st->beta[c] = beta;
                st->alpha[c] = a; st->neg_alpha[c] = -a;
                st->rho[c] = v[c];
            }
        }
        const int anybad = __syncthreads_or(bad);
        if (threadIdx.x == 0) {
            const int stop = all || anybad || st->it >= st->max_iters;
            st->stop = stop;
            // the remaining products of this iteration only feed the next one
            st->skip = stop ? 1 : 0;
            st->nodrift = (!anybad && (st->it % 20 == 0 || all)) ? 0 : 1;
            if (anybad) st->err = MRS_ERR_BREAKDOWN;
            set_loop(st, !stop);
        }
        return;
    }
    case EPI_PBICG_DRIFT: {
        // solvers.py:415-423: ||r_init - op(zacc)|| / max(rnorm, tiny) > limit
        bool drift = false;
        if (act) {
            const double rec = st->rnorm[c] > 2.2250738585072014e-308 ? st->rnorm[c]
                                                                        : 2.2250738585072014e-308;
            drift = divd(sqrt(v[c]), rec) > st->drift_limit;
        }
        if (__syncthreads_or(drift) && threadIdx.x == 0) {
            st->err = MRS_ERR_INSTABILITY;
            st->stop = 1;
            st->skip = 1;
            set_loop(st, false);
        }
        return;
    }
    }
    int anybad = __syncthreads_or(bad);
    if (anybad && threadIdx.x == 0) {
        st->err = MRS_ERR_BREAKDOWN;
        st->skip = 1;
        st->stop = 1;
        st->pskip = 1;
        st->nodrift = 1;
        set_loop(st, false);
    }
}

// Finish a reduction whose per-CTA partial (Km values) sits in smem `blk`.
// All threads of every CTA call this.
static __device__ void finish_reduction(const RedArgs& ra, const double* blk, int Km, int m) {
    __shared__ bool s_last;
    __shared__ double s_out[kMaxK * kMaxM];
    const int G = gridDim.x;
    // value-major partials [Km][G]: the last CTA reads each value's G partials
    // with coalesced warp loads
    for (int i = threadIdx.x; i < Km; i += blockDim.x)
        ra.partials[(size_t)i * G + blockIdx.x] = blk[i];
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned t = atomicAdd(ra.ticket, 1u);
        MRS_DCHECK(t < (unsigned)G);           // a stale or shared ticket overshoots
        s_last = (t == (unsigned)G - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // warp w folds values j = w, w + nw, ...: lane l sums partials
    // b = l, l + 32, ... (loads batched 8 deep), then a fixed xor tree.
    // Shape depends only on (Km, G): deterministic.
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int j = warp; j < Km; j += nw) {
        const double* p = ra.partials + (size_t)j * G;
        double acc = 0.0;
        int b = lane;
        for (; b + 7 * 32 < G; b += 8 * 32) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldcg(p + b + u * 32);
#pragma unroll
            for (int u = 0; u < 8; ++u) acc = add(acc, v[u]);
        }
        for (; b < G; b += 32) acc = add(acc, __ldcg(p + b));
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc = add(acc, __shfl_xor_sync(0xffffffffu, acc, off));
        if (lane == 0) {
            s_out[j] = acc;
            if (ra.out) ra.out[j] = acc;
        }
    }
    if (threadIdx.x == 0) *ra.ticket = 0u;
    __syncthreads();
    if (ra.epi != EPI_NONE) run_epilogue(ra.epi, ra.st, s_out, m);
}

}  // namespace mrs
