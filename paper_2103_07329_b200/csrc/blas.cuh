// blas.cuh -- blocked multi-RHS vector kernels with per-column scalars and
// fused reductions (reference src/blas.py:107-292, _ckernels.pyx:82-162),
// plus the solver-specific fused updates the Krylov drivers use.
//
// Layout: a CTA of 256 threads covers RPB = 256 / m rows; thread t owns
// column c = t % m for all its rows, so per-column scalars (alpha_j, beta_j,
// ...) are loaded once per thread and every global access is a coalesced
// 8-byte access of consecutive elements.  Rows are unrolled 4 deep for
// memory-level parallelism.  Each element uses exactly the reference's
// expression (separately rounded mul/add).
#pragma once

#include "reduce.cuh"

namespace mrs {

enum VecOp : int {
    V_AXPBY = 0,      // y = b*y + a*x                          (axpby)
    V_ADD2,           // y = (y + a*u) + b*v                    (add2_scaled)
    V_PAIRED,         // y1 = (y1 + a*u) + b*s; y2 = s - c*w    (fused_paired_update)
    V_DOT,            // sum x*y                                (dot_partial)
    V_UPDATE_DOT,     // t = b*y + a*x; y = t; sum t*t          (fused_update_dot)
    V_UPDATE_DOT2,    // t = u - c*w; y = t; sum z*t, sum t*t   (fused_update_dot2)
    V_COPY,           // y = x
    V_CG_UPDATE,      // x += a*p; r += na*q; sum r*r          (cg_solve:176-178)
    V_CG_UPDATE_JAC,  // ... and z = w*(r/d); sum r*z          (+ Jacobi preconditioner)
    V_P_UPDATE,       // p = b*p + z                            (cg_solve:185)
    V_SEED,           // y = seed(x): w*(x/d) or x/(d*theta)     (zero-guess first smoother step)
    V_BICG_P,         // p = beta*(p + nw*v) + r                (bicgstab:250-251)
    V_BICG_S,         // s = r + na*v                           (bicgstab:262-263)
    V_DOT3,           // (t.s, t.t, s.s)                        (bicgstab:271 + :273)
    V_BICG_XR,        // X = (X + a*ph) + w*sh; r = s + nw*t; (r0.r, r.r)  (bicgstab:285-288)
    V_DOT2,           // (x.y, u.v)
};

template <int OP> struct VK { static constexpr int K = 0; };
template <> struct VK<V_DOT> { static constexpr int K = 1; };
template <> struct VK<V_UPDATE_DOT> { static constexpr int K = 1; };
template <> struct VK<V_UPDATE_DOT2> { static constexpr int K = 2; };
template <> struct VK<V_CG_UPDATE> { static constexpr int K = 1; };
template <> struct VK<V_CG_UPDATE_JAC> { static constexpr int K = 2; };
template <> struct VK<V_DOT3> { static constexpr int K = 3; };
template <> struct VK<V_BICG_XR> { static constexpr int K = 2; };
template <> struct VK<V_DOT2> { static constexpr int K = 2; };

struct VArgs {
    int64_t n, m;
    double* y; double* y2; double* y3;
    const double* x; const double* u; const double* v; const double* w; const double* z;
    const double* s;
    const double* a; const double* b; const double* c;    // per-column scalars (device)
    const double* d;                                       // per-row diagonal
    double wt, theta;                                      // Jacobi weight / Chebyshev theta
    const int* guard;
    const int* guard_it;     // V_BICG_P: no-op while *guard_it == 0 (first iteration)
    int seed;                // 1/2: also write seed_out = seed(produced vector) (spmm.cuh)
    double* seed_out;
    const double* seed_d;
    double seed_w;           // Jacobi weight or Chebyshev theta
    RedArgs red;
};

// Block-level column reduction of K per-thread accumulators; result in blk[K*m].
template <int K>
__device__ __forceinline__ void block_reduce_cols(double (&acc)[K], int m, double* blk) {
    const int nw = kThreads / 32;
    if (m <= 32 && (32 % m) == 0) {
        __shared__ double s_w[kThreads / 32][K > 0 ? K * 32 : 1];
#pragma unroll
        for (int off = m; off < 32; off <<= 1)
#pragma unroll
            for (int k = 0; k < K; ++k)
                acc[k] = add(acc[k], __shfl_xor_sync(0xffffffffu, acc[k], off));
        const int warp = threadIdx.x / 32, wl = threadIdx.x % 32;
        if (wl < m)
#pragma unroll
            for (int k = 0; k < K; ++k) s_w[warp][k * m + wl] = acc[k];
        __syncthreads();
        if (threadIdx.x < K * m) {
            double t = s_w[0][threadIdx.x];
            for (int w = 1; w < nw; ++w) t = add(t, s_w[w][threadIdx.x]);
            blk[threadIdx.x] = t;
        }
    } else {
        __shared__ double s_t[K > 0 ? K : 1][kThreads];
        const int rpb = kThreads / m;
#pragma unroll
        for (int k = 0; k < K; ++k) s_t[k][threadIdx.x] = acc[k];
        __syncthreads();
        if (threadIdx.x < K * m) {
            const int k = threadIdx.x / m, c = threadIdx.x % m;
            double t = s_t[k][c];
            for (int r = 1; r < rpb; ++r) t = add(t, s_t[k][r * m + c]);
            blk[threadIdx.x] = t;
        }
    }
    __syncthreads();
}

// Zero-guess smoother seed of a produced value v at row i (spmm.cuh seed_value).
__device__ __forceinline__ double seed_of(const VArgs& A, double v, int64_t i) {
    const double d = __ldg(A.seed_d + i);
    return A.seed == 1 ? mul(A.seed_w, divd(v, d)) : divd(v, mul(d, A.seed_w));
}

template <int OP>
__device__ __forceinline__ void vec_elem(const VArgs& A, int64_t i, int64_t e, int c,
                                         double sa, double sb, double sc,
                                         double (&acc)[VK<OP>::K > 0 ? VK<OP>::K : 1]) {
    if constexpr (OP == V_AXPBY) {
        A.y[e] = add(mul(sb, A.y[e]), mul(sa, __ldg(A.x + e)));
    } else if constexpr (OP == V_ADD2) {
        A.y[e] = add(add(A.y[e], mul(sa, __ldg(A.u + e))), mul(sb, __ldg(A.v + e)));
    } else if constexpr (OP == V_PAIRED) {
        double sv = __ldg(A.s + e);
        A.y[e] = add(add(A.y[e], mul(sa, __ldg(A.u + e))), mul(sb, sv));
        A.y2[e] = sub(sv, mul(sc, __ldg(A.w + e)));
    } else if constexpr (OP == V_DOT) {
        acc[0] = add(acc[0], mul(__ldg(A.x + e), __ldg(A.z + e)));
    } else if constexpr (OP == V_UPDATE_DOT) {
        double t = add(mul(sb, A.y[e]), mul(sa, __ldg(A.x + e)));
        A.y[e] = t;
        acc[0] = add(acc[0], mul(t, t));
    } else if constexpr (OP == V_UPDATE_DOT2) {
        double t = sub(A.u[e], mul(sc, A.w[e]));   // y may alias u or w: plain loads
        A.y[e] = t;
        acc[0] = add(acc[0], mul(__ldg(A.z + e), t));
        acc[1] = add(acc[1], mul(t, t));
    } else if constexpr (OP == V_COPY) {
        const double v = __ldg(A.x + e);
        A.y[e] = v;
        if (A.seed) A.seed_out[e] = seed_of(A, v, i);
    } else if constexpr (OP == V_CG_UPDATE || OP == V_CG_UPDATE_JAC) {
        // X = 1*X + alpha*p ; r = 1*r + (-alpha)*q   (axpby, blas.py:144)
        A.y[e] = add(A.y[e], mul(sa, __ldg(A.x + e)));
        double r = add(A.y2[e], mul(sb, __ldg(A.u + e)));
        A.y2[e] = r;
        acc[0] = add(acc[0], mul(r, r));
        if (A.seed) A.seed_out[e] = seed_of(A, r, i);
        if constexpr (OP == V_CG_UPDATE_JAC) {
            // z = 0 + w*(r/d) (jacobi_sweep from a zero guess, blas2.py:181)
            double zz = mul(A.wt, divd(r, __ldg(A.d + i)));
            A.y3[e] = zz;
            acc[1] = add(acc[1], mul(r, zz));
        }
    } else if constexpr (OP == V_P_UPDATE) {
        A.y[e] = add(mul(sb, A.y[e]), __ldg(A.x + e));
    } else if constexpr (OP == V_SEED) {
        A.y[e] = seed_of(A, __ldg(A.x + e), i);
    } else if constexpr (OP == V_BICG_P) {
        // p -= omega v ; p = r + beta p  (two axpby passes fused, same rounding)
        double t = add(A.y[e], mul(sc, __ldg(A.v + e)));
        double p = add(mul(sb, t), __ldg(A.x + e));
        A.y[e] = p;
        if (A.seed) A.seed_out[e] = seed_of(A, p, i);
    } else if constexpr (OP == V_BICG_S) {
        double s = add(__ldg(A.x + e), mul(sa, __ldg(A.v + e)));
        A.y[e] = s;
        if (A.seed) A.seed_out[e] = seed_of(A, s, i);
    } else if constexpr (OP == V_DOT3) {
        double t = __ldg(A.x + e), s = __ldg(A.s + e);
        acc[0] = add(acc[0], mul(t, s));
        acc[1] = add(acc[1], mul(t, t));
        acc[2] = add(acc[2], mul(s, s));
    } else if constexpr (OP == V_BICG_XR) {
        // add2_scaled(X, alpha, ph, omega, sh); r = s ; axpby(-omega, t, 1, r)
        A.y[e] = add(add(A.y[e], mul(sa, __ldg(A.u + e))), mul(sb, __ldg(A.v + e)));
        double r = add(__ldg(A.s + e), mul(sc, __ldg(A.w + e)));
        A.y2[e] = r;
        acc[0] = add(acc[0], mul(__ldg(A.z + e), r));
        acc[1] = add(acc[1], mul(r, r));
    } else if constexpr (OP == V_DOT2) {
        acc[0] = add(acc[0], mul(__ldg(A.x + e), __ldg(A.z + e)));
        acc[1] = add(acc[1], mul(__ldg(A.u + e), __ldg(A.v + e)));
    }
}

template <int OP>
__global__ void __launch_bounds__(kThreads) vec_kernel(VArgs A) {
    if (A.guard && *A.guard) return;
    if constexpr (OP == V_BICG_P) {
        if (A.guard_it && *A.guard_it == 0) return;
    }
    constexpr int K = VK<OP>::K;
    constexpr int U = 4;
    const int m = (int)A.m;
    const int rpb = kThreads / m;
    const int c = threadIdx.x % m;
    const int rs = threadIdx.x / m;
    double acc[K > 0 ? K : 1];
#pragma unroll
    for (int k = 0; k < (K > 0 ? K : 1); ++k) acc[k] = 0.0;
    double sa = 0.0, sb = 0.0, sc = 0.0;
    if (rs < rpb) {
        if (A.a) sa = __ldg(A.a + c);
        if (A.b) sb = __ldg(A.b + c);
        if (A.c) sc = __ldg(A.c + c);
        const int64_t chunk = (int64_t)rpb * U;
        for (int64_t base = (int64_t)blockIdx.x * chunk; base < A.n;
             base += (int64_t)gridDim.x * chunk) {
#pragma unroll
            for (int j = 0; j < U; ++j) {
                int64_t i = base + rs + (int64_t)j * rpb;
                if (i < A.n) vec_elem<OP>(A, i, i * m + c, c, sa, sb, sc, acc);
            }
        }
    }
    if constexpr (K > 0) {
        __shared__ double s_blk[K * kMaxM];
        block_reduce_cols<K>(acc, m, s_blk);
        finish_reduction(A.red, s_blk, K * m, m);
    }
}

}  // namespace mrs
