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
    // reordered BiCGStab (solvers.py:296-364)
    V_DOT5,           // (t.s, t.t, r0.s, r0.t, s.s)            (rbicgstab:336-338)
    V_BICG_XR0,       // X = (X + a*ph) + w*sh; r = s + nw*t     (rbicgstab:345-351, no dots)
    // pipelined BiCGStab (solvers.py:367-479)
    V_PBICG_QY,       // (it > 1) p,s,z = r,w,t + beta*(p,s,z - omega*(s,z,v));
                      // q = r + na*s; y = w + na*z; (q.y, y.y)  (pbicgstab:432-443)
    V_PBICG_W,        // t += na*v; w = y + nw*t;
                      // (r0.r, r0.w, r0.s, r0.z, r.r)        (pbicgstab:452-458, 461-463)
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
template <> struct VK<V_DOT5> { static constexpr int K = 5; };
template <> struct VK<V_PBICG_QY> { static constexpr int K = 2; };
template <> struct VK<V_PBICG_W> { static constexpr int K = 5; };

// Operand roles of the pipelined-BiCGStab kernels (the fields are generic):
//   V_PBICG_QY: y=p y2=s y3=z (read+write), y4=q y5=y (write), x=r w=w u=t v=v;
//               a=-alpha b=beta c=-omega, guard_it=&it (it == 0: no p/s/z update)
//   V_PBICG_W:  y=t (read+write), y2=w (write), x=v u=y z=r0 v=r s=s w=z;
//               a=-alpha c=-omega
struct VArgs {
    int64_t n, m;
    double* y; double* y2; double* y3; double* y4; double* y5;
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

// Zero-guess smoother seed of a produced value v with row diagonal d
// (spmm.cuh seed_value).
__device__ __forceinline__ double seed_of(const VArgs& A, double v, double d) {
    if (A.seed == 3) return 0.0;                       // Gauss-Seidel: x = 0
    return A.seed == 1 ? mul(A.seed_w, divd(v, d)) : divd(v, mul(d, A.seed_w));
}

// Operands of one element, loaded before any store of the unrolled group so
// the loads of U rows overlap (outputs may alias inputs element-wise).
struct Ld { double y, y2, y3, x, u, v, w, z, s, d; };

template <int OP> struct Uses {
    static constexpr bool y = OP == V_AXPBY || OP == V_ADD2 || OP == V_PAIRED || OP == V_UPDATE_DOT ||
                              OP == V_CG_UPDATE || OP == V_CG_UPDATE_JAC || OP == V_P_UPDATE ||
                              OP == V_BICG_P || OP == V_BICG_XR || OP == V_BICG_XR0 ||
                              OP == V_PBICG_QY || OP == V_PBICG_W;
    static constexpr bool y2 = OP == V_CG_UPDATE || OP == V_CG_UPDATE_JAC || OP == V_PBICG_QY;
    static constexpr bool y3 = OP == V_PBICG_QY;
    static constexpr bool x = OP == V_AXPBY || OP == V_DOT || OP == V_UPDATE_DOT || OP == V_COPY ||
                              OP == V_CG_UPDATE || OP == V_CG_UPDATE_JAC || OP == V_P_UPDATE ||
                              OP == V_SEED || OP == V_BICG_P || OP == V_BICG_S || OP == V_DOT3 ||
                              OP == V_DOT2 || OP == V_DOT5 || OP == V_PBICG_QY || OP == V_PBICG_W;
    static constexpr bool u = OP == V_ADD2 || OP == V_PAIRED || OP == V_UPDATE_DOT2 ||
                              OP == V_CG_UPDATE || OP == V_CG_UPDATE_JAC || OP == V_BICG_XR ||
                              OP == V_DOT2 || OP == V_BICG_XR0 || OP == V_PBICG_QY ||
                              OP == V_PBICG_W;
    static constexpr bool v = OP == V_ADD2 || OP == V_BICG_P || OP == V_BICG_S || OP == V_BICG_XR ||
                              OP == V_DOT2 || OP == V_BICG_XR0 || OP == V_PBICG_QY ||
                              OP == V_PBICG_W;
    static constexpr bool w = OP == V_PAIRED || OP == V_UPDATE_DOT2 || OP == V_BICG_XR ||
                              OP == V_BICG_XR0 || OP == V_PBICG_QY || OP == V_PBICG_W;
    static constexpr bool z = OP == V_DOT || OP == V_UPDATE_DOT2 || OP == V_BICG_XR || OP == V_DOT2 ||
                              OP == V_DOT5 || OP == V_PBICG_W;
    static constexpr bool s = OP == V_PAIRED || OP == V_DOT3 || OP == V_BICG_XR || OP == V_DOT5 ||
                              OP == V_BICG_XR0 || OP == V_PBICG_W;
    static constexpr bool d = OP == V_CG_UPDATE_JAC || OP == V_SEED;   // + any seeding op
};

template <int OP>
__device__ __forceinline__ void vec_load(const VArgs& A, int64_t e, int64_t i, Ld& L) {
    using Us = Uses<OP>;
    if constexpr (Us::y) L.y = A.y[e];
    if constexpr (Us::y2) L.y2 = A.y2[e];
    if constexpr (Us::y3) L.y3 = A.y3[e];
    if constexpr (Us::x) L.x = __ldg(A.x + e);
    if constexpr (Us::u) L.u = A.u[e];
    if constexpr (Us::v) L.v = __ldg(A.v + e);
    if constexpr (Us::w) L.w = A.w[e];
    if constexpr (Us::z) L.z = __ldg(A.z + e);
    if constexpr (Us::s) L.s = __ldg(A.s + e);
    if constexpr (Us::d) L.d = __ldg((OP == V_CG_UPDATE_JAC ? A.d : A.seed_d) + i);
    else if (A.seed) L.d = __ldg(A.seed_d + i);
}

template <int OP>
__device__ __forceinline__ void vec_compute(const VArgs& A, int64_t e, const Ld& L,
                                            double sa, double sb, double sc, bool first,
                                            double (&acc)[VK<OP>::K > 0 ? VK<OP>::K : 1]) {
    if constexpr (OP == V_AXPBY) {
        A.y[e] = add(mul(sb, L.y), mul(sa, L.x));
    } else if constexpr (OP == V_ADD2) {
        A.y[e] = add(add(L.y, mul(sa, L.u)), mul(sb, L.v));
    } else if constexpr (OP == V_PAIRED) {
        A.y[e] = add(add(L.y, mul(sa, L.u)), mul(sb, L.s));
        A.y2[e] = sub(L.s, mul(sc, L.w));
    } else if constexpr (OP == V_DOT) {
        acc[0] = add(acc[0], mul(L.x, L.z));
    } else if constexpr (OP == V_UPDATE_DOT) {
        const double t = add(mul(sb, L.y), mul(sa, L.x));
        A.y[e] = t;
        acc[0] = add(acc[0], mul(t, t));
    } else if constexpr (OP == V_UPDATE_DOT2) {
        const double t = sub(L.u, mul(sc, L.w));
        A.y[e] = t;
        acc[0] = add(acc[0], mul(L.z, t));
        acc[1] = add(acc[1], mul(t, t));
    } else if constexpr (OP == V_COPY) {
        A.y[e] = L.x;
        if (A.seed) A.seed_out[e] = seed_of(A, L.x, L.d);
    } else if constexpr (OP == V_CG_UPDATE || OP == V_CG_UPDATE_JAC) {
        // X = 1*X + alpha*p ; r = 1*r + (-alpha)*q   (axpby, blas.py:144)
        A.y[e] = add(L.y, mul(sa, L.x));
        const double r = add(L.y2, mul(sb, L.u));
        A.y2[e] = r;
        acc[0] = add(acc[0], mul(r, r));
        if constexpr (OP == V_CG_UPDATE_JAC) {
            // z = 0 + w*(r/d) (jacobi_sweep from a zero guess, blas2.py:181)
            const double zz = mul(A.wt, divd(r, L.d));
            A.y3[e] = zz;
            acc[1] = add(acc[1], mul(r, zz));
        } else {
            if (A.seed) A.seed_out[e] = seed_of(A, r, L.d);
        }
    } else if constexpr (OP == V_P_UPDATE) {
        A.y[e] = add(mul(sb, L.y), L.x);
    } else if constexpr (OP == V_SEED) {
        A.y[e] = seed_of(A, L.x, L.d);
    } else if constexpr (OP == V_BICG_P) {
        // p -= omega v ; p = r + beta p  (two axpby passes fused, same rounding)
        const double t = add(L.y, mul(sc, L.v));
        const double p = add(mul(sb, t), L.x);
        A.y[e] = p;
        if (A.seed) A.seed_out[e] = seed_of(A, p, L.d);
    } else if constexpr (OP == V_BICG_S) {
        const double s = add(L.x, mul(sa, L.v));
        A.y[e] = s;
        if (A.seed) A.seed_out[e] = seed_of(A, s, L.d);
    } else if constexpr (OP == V_DOT3) {
        acc[0] = add(acc[0], mul(L.x, L.s));
        acc[1] = add(acc[1], mul(L.x, L.x));
        acc[2] = add(acc[2], mul(L.s, L.s));
    } else if constexpr (OP == V_BICG_XR) {
        // add2_scaled(X, alpha, ph, omega, sh); r = s ; axpby(-omega, t, 1, r)
        A.y[e] = add(add(L.y, mul(sa, L.u)), mul(sb, L.v));
        const double r = add(L.s, mul(sc, L.w));
        A.y2[e] = r;
        acc[0] = add(acc[0], mul(L.z, r));
        acc[1] = add(acc[1], mul(r, r));
    } else if constexpr (OP == V_DOT2) {
        acc[0] = add(acc[0], mul(L.x, L.z));
        acc[1] = add(acc[1], mul(L.u, L.v));
    } else if constexpr (OP == V_DOT5) {
        // dot_many([(t, s), (t, t), (r0, s), (r0, t), (s, s)]): x=t s=s z=r0
        acc[0] = add(acc[0], mul(L.x, L.s));
        acc[1] = add(acc[1], mul(L.x, L.x));
        acc[2] = add(acc[2], mul(L.z, L.s));
        acc[3] = add(acc[3], mul(L.z, L.x));
        acc[4] = add(acc[4], mul(L.s, L.s));
    } else if constexpr (OP == V_BICG_XR0) {
        A.y[e] = add(add(L.y, mul(sa, L.u)), mul(sb, L.v));
        A.y2[e] = add(L.s, mul(sc, L.w));
    } else if constexpr (OP == V_PBICG_QY) {
        double p = L.y, s = L.y2, z = L.y3;
        if (!first) {
            // axpby(-omega, s, 1, p); axpby(1, r, beta, p) and the same for s, z
            p = add(mul(sb, add(p, mul(sc, s))), L.x);
            s = add(mul(sb, add(s, mul(sc, z))), L.w);
            z = add(mul(sb, add(z, mul(sc, L.v))), L.u);
            A.y[e] = p; A.y2[e] = s; A.y3[e] = z;
        }
        const double q = add(L.x, mul(sa, s));       // q = r - alpha s
        const double yv = add(L.w, mul(sa, z));      // y = w - alpha z
        A.y4[e] = q; A.y5[e] = yv;
        acc[0] = add(acc[0], mul(q, yv));
        acc[1] = add(acc[1], mul(yv, yv));
        if (A.seed) A.seed_out[e] = seed_of(A, z, L.d);
    } else if constexpr (OP == V_PBICG_W) {
        const double t = add(L.y, mul(sa, L.x));     // t -= alpha v
        const double w = add(L.u, mul(sc, t));       // w = y - omega t
        A.y[e] = t; A.y2[e] = w;
        acc[0] = add(acc[0], mul(L.z, L.v));         // (r0, r)
        acc[1] = add(acc[1], mul(L.z, w));           // (r0, w)
        acc[2] = add(acc[2], mul(L.z, L.s));         // (r0, s)
        acc[3] = add(acc[3], mul(L.z, L.w));         // (r0, z)
        acc[4] = add(acc[4], mul(L.v, L.v));         // (r, r)
        if (A.seed) A.seed_out[e] = seed_of(A, w, L.d);
    }
}

constexpr int kVecUnroll = 4;
// rows in flight per thread: fewer for the operand-heavy fused updates so
// they stay spill-free under the 64-register cap (4 CTAs/SM)
template <int OP> __host__ __device__ constexpr int vec_unroll() {
    using Us = Uses<OP>;
    constexpr int ops = Us::y + Us::y2 + Us::y3 + Us::x + Us::u + Us::v + Us::w + Us::z + Us::s;
    return ops >= 7 ? 1 : ops >= 4 ? 2 : kVecUnroll;
}

// CTA b owns the contiguous row range [b*chunk, (b+1)*chunk) (chunk a multiple
// of RPB*U); thread (rs, c) handles column c of rows rs, rs + RPB, ...
template <int OP>
__global__ void __launch_bounds__(kThreads, 4) vec_kernel(VArgs A, int64_t chunk) {
    pdl_enter();
    if (A.guard && *A.guard) return;
    if constexpr (OP == V_BICG_P) {
        if (A.guard_it && *A.guard_it == 0) return;
    }
    constexpr int K = VK<OP>::K;
    constexpr int U = vec_unroll<OP>();
    const int m = (int)A.m;
    const int rpb = kThreads / m;
    const int c = threadIdx.x % m;
    const int rs = threadIdx.x / m;
    double acc[K > 0 ? K : 1];
#pragma unroll
    for (int k = 0; k < (K > 0 ? K : 1); ++k) acc[k] = 0.0;
    const bool first = A.guard_it && *A.guard_it == 0;   // V_PBICG_QY
    if (rs < rpb) {
        const double sa = A.a ? __ldg(A.a + c) : 0.0;
        const double sb = A.b ? __ldg(A.b + c) : 0.0;
        const double sc = A.c ? __ldg(A.c + c) : 0.0;
        const int64_t r0 = (int64_t)blockIdx.x * chunk;
        const int64_t r1 = min(r0 + chunk, A.n);
        for (int64_t base = r0; base < r1; base += (int64_t)rpb * U) {
            Ld L[U];
#pragma unroll
            for (int j = 0; j < U; ++j) {
                const int64_t i = base + rs + (int64_t)j * rpb;
                if (i < r1) vec_load<OP>(A, i * m + c, i, L[j]);
            }
            compiler_fence();
#pragma unroll
            for (int j = 0; j < U; ++j) {
                const int64_t i = base + rs + (int64_t)j * rpb;
                if (i < r1) vec_compute<OP>(A, i * m + c, L[j], sa, sb, sc, first, acc);
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
