// band_probe.cu -- standalone A/B of SpMM designs for banded-random operators
// (BASELINE config 5: n = 2^22, ~16 entries/row, columns within +-4096 of the
// diagonal).  Not part of the library.  Every variant is checked bitwise
// against the lane kernel (the library's round-1/2 design).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
//        -o band_probe band_probe.cu && ./band_probe [m] [n_log2]
//
// Variants:
//   lane    : LPR lanes per row, chunks of 64 rows strided over the grid (library kernel)
//   remap   : same kernel, each SM walks ONE contiguous row range (its CTAs interleave
//             64-row chunks inside it): the gathered x window of the SM's rows is reused
//             from L1 instead of L2; optional no-allocate matrix stream
//   stream  : m in {1, 2}: the CTA's whole x window in shared memory (TMA bulk copy),
//             entry-parallel products into shared memory (coalesced matrix stream),
//             then one thread per row adds its products in entry order
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <random>
#include <string>
#include <vector>

#define CK(x)                                                                        \
    do {                                                                             \
        cudaError_t e = (x);                                                         \
        if (e != cudaSuccess) {                                                      \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
            exit(1);                                                                 \
        }                                                                            \
    } while (0)

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ void fence() { asm volatile("" ::: "memory"); }

template <int M> struct Lay {
    static constexpr int CPL = (M == 1) ? 1 : 2;
    static constexpr int LPR = M / CPL;
};

struct Args {
    const int* rp;
    const uint32_t* ci;
    const double* v;
    int n;
    const double* x;
    double* y;
    int chunk;
    int nsm;          // remap: SMs
    int cps;          // remap: CTAs per SM
    int band;         // max |col - row|
    int R;            // stream: rows per CTA block
    int nblocks;
};

template <int CPL> struct V { double v[CPL]; };
template <int CPL> __device__ __forceinline__ V<CPL> ldx(const double* p) {
    V<CPL> r;
    if constexpr (CPL == 1) r.v[0] = __ldg(p);
    else {
#pragma unroll
        for (int i = 0; i < CPL; i += 2) {
            double2 t = __ldg(reinterpret_cast<const double2*>(p + i));
            r.v[i] = t.x; r.v[i + 1] = t.y;
        }
    }
    return r;
}
template <int CPL> __device__ __forceinline__ void stv(double* p, const V<CPL>& a) {
    if constexpr (CPL == 1) *p = a.v[0];
    else {
#pragma unroll
        for (int i = 0; i < CPL; i += 2)
            *reinterpret_cast<double2*>(p + i) = make_double2(a.v[i], a.v[i + 1]);
    }
}
__device__ __forceinline__ uint32_t ld_na_u32(const uint32_t* p) {
    uint32_t r;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ double ld_na_f64(const double* p) {
    double r;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
    return r;
}

// one row of the lane kernel (ASSIGN): entries in groups of UNR
template <int M, int UNR, int NA>
__device__ __forceinline__ void lane_row(const Args& a, int row, int cofs) {
    constexpr int CPL = Lay<M>::CPL;
    const int lo = __ldg(a.rp + row), hi = __ldg(a.rp + row + 1);
    const int o = row * M + cofs;
    V<CPL> acc;
#pragma unroll
    for (int i = 0; i < CPL; ++i) acc.v[i] = 0.0;
    for (int k = lo; k < hi; k += UNR) {
        int c[UNR]; double v[UNR]; V<CPL> g[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const int kk = (k + u < hi) ? k + u : lo;
            if (NA) { c[u] = (int)ld_na_u32(a.ci + kk); v[u] = ld_na_f64(a.v + kk); }
            else { c[u] = (int)__ldg(a.ci + kk); v[u] = __ldg(a.v + kk); }
        }
        fence();
#pragma unroll
        for (int u = 0; u < UNR; ++u) g[u] = ldx<CPL>(a.x + c[u] * M + cofs);
        fence();
#pragma unroll
        for (int u = 0; u < UNR; ++u)
            if (k + u < hi)
#pragma unroll
                for (int i = 0; i < CPL; ++i) acc.v[i] = add(acc.v[i], mul(v[u], g[u].v[i]));
    }
    stv<CPL>(a.y + o, acc);
}

template <int M, int UNR, int MINB>
__global__ void __launch_bounds__(256, MINB) k_lane(Args a) {
    constexpr int CPL = Lay<M>::CPL, LPR = Lay<M>::LPR, RPB = 256 / LPR;
    const int cofs = (threadIdx.x % LPR) * CPL;
    for (int r0 = blockIdx.x * a.chunk; r0 < a.n; r0 += gridDim.x * a.chunk) {
        const int r1 = min(r0 + a.chunk, a.n);
        for (int row = r0 + threadIdx.x / LPR; row < r1; row += RPB) lane_row<M, UNR, 0>(a, row, cofs);
    }
}

// remap: CTA b belongs to "SM slot" s = b % nsm, sub-slot q = b / nsm; slot s owns
// rows [s*per, (s+1)*per); its cps CTAs take chunks q, q + cps, ... of that range.
template <int M, int UNR, int MINB, int NA>
__global__ void __launch_bounds__(256, MINB) k_remap(Args a) {
    constexpr int CPL = Lay<M>::CPL, LPR = Lay<M>::LPR, RPB = 256 / LPR;
    const int cofs = (threadIdx.x % LPR) * CPL;
    const int s = blockIdx.x % a.nsm, q = blockIdx.x / a.nsm;
    const long per = ((long)a.n + a.nsm - 1) / a.nsm;
    const int rs = (int)min((long)a.n, s * per), re = (int)min((long)a.n, (s + 1) * per);
    for (int r0 = rs + q * a.chunk; r0 < re; r0 += a.cps * a.chunk) {
        const int r1 = min(r0 + a.chunk, re);
        for (int row = r0 + threadIdx.x / LPR; row < r1; row += RPB) lane_row<M, UNR, NA>(a, row, cofs);
    }
}

// ------------------------------------------------------------------ stream (m = 1, 2)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mb_init(uint64_t* b, int cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx)
                 : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra W;\n}" ::"r"(smem_u32(b)), "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// CTA = one block of R consecutive rows (strided over the grid).  smem: x window
// (band + R + band rows) | products PE x M | barrier.
template <int M, int T, int PE, int UNR>
__global__ void __launch_bounds__(T) k_stream(Args a) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int WR = a.R + 2 * a.band + 2;                 // window rows (capacity)
    double* xs = reinterpret_cast<double*>(sm);
    double* P = xs + (size_t)WR * M;
    uint64_t* bar = reinterpret_cast<uint64_t*>(P + (size_t)PE * M);
    if (threadIdx.x == 0) {
        mb_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t phase = 0;
    for (int blk = blockIdx.x; blk < a.nblocks; blk += gridDim.x) {
        const int r0 = blk * a.R, r1 = min(r0 + a.R, a.n);
        int wlo = max(0, r0 - a.band);
        if (M == 1) wlo &= ~1;                           // 16-byte aligned source
        const int whi = min(a.n, r1 + a.band);
        const int wn = whi - wlo;
        if (threadIdx.x == 0) {
            // (all threads passed the previous block's last __syncthreads: xs is free)
            const uint32_t bytes = (uint32_t)((size_t)wn * M * 8) & ~15u;
            mb_expect(bar, bytes);
            uint32_t off = 0;
            while (off < bytes) {
                const uint32_t pc = min(bytes - off, 32768u);
                bulk_g2s(reinterpret_cast<unsigned char*>(xs) + off,
                         reinterpret_cast<const unsigned char*>(a.x + (size_t)wlo * M) + off, pc, bar);
                off += pc;
            }
            if (((size_t)wn * M * 8) & 15) xs[(size_t)wn * M - 1] = a.x[(size_t)whi * M - 1];
        }
        mb_wait(bar, phase);
        phase ^= 1;
        __syncthreads();       // also publishes thread 0's tail element
        for (int rb = r0; rb < r1; rb += T) {            // sub-block: one row per thread
            const int re = min(rb + T, r1);
            const int row = rb + threadIdx.x;
            const int eb = __ldg(a.rp + rb), ee = __ldg(a.rp + re);
            int lo = 0, hi = 0;
            if (row < re) { lo = __ldg(a.rp + row); hi = __ldg(a.rp + row + 1); }
            double acc[M];
#pragma unroll
            for (int i = 0; i < M; ++i) acc[i] = 0.0;
            for (int pb = eb; pb < ee; pb += PE) {       // pieces of PE entries (usually one)
                const int cnt = min(PE, ee - pb);
                // phase 1: products, entry-parallel, UNR loads in flight per thread
                for (int i0 = threadIdx.x; i0 < cnt; i0 += T * UNR) {
                    int c[UNR]; double v[UNR];
#pragma unroll
                    for (int u = 0; u < UNR; ++u) {
                        const int i = i0 + u * T;
                        const int e = pb + (i < cnt ? i : 0);
                        c[u] = (int)ld_na_u32(a.ci + e);
                        v[u] = ld_na_f64(a.v + e);
                    }
                    fence();
#pragma unroll
                    for (int u = 0; u < UNR; ++u) {
                        const int i = i0 + u * T;
                        if (i < cnt) {
                            const double* xr = xs + (size_t)(c[u] - wlo) * M;
                            if constexpr (M == 1) P[i] = mul(v[u], xr[0]);
                            else {
                                const double2 t = *reinterpret_cast<const double2*>(xr);
                                *reinterpret_cast<double2*>(P + 2 * i) = make_double2(mul(v[u], t.x), mul(v[u], t.y));
                            }
                        }
                    }
                }
                __syncthreads();
                // phase 2: the row's products of this piece, in entry order
                const int klo = max(lo, pb) - pb, khi = min(hi, pb + cnt) - pb;
                for (int k = klo; k < khi; ++k) {
                    if constexpr (M == 1) acc[0] = add(acc[0], P[k]);
                    else {
                        const double2 t = *reinterpret_cast<const double2*>(P + 2 * k);
                        acc[0] = add(acc[0], t.x); acc[1] = add(acc[1], t.y);
                    }
                }
                __syncthreads();
            }
            if (row < re) {
                if constexpr (M == 1) a.y[row] = acc[0];
                else *reinterpret_cast<double2*>(a.y + 2 * (size_t)row) = make_double2(acc[0], acc[1]);
            }
        }
    }
}



// ------------------------------------------------------------------ stream2 (m = 1, 2)
// TMA-fed: a producer warp streams the CSR entries (columns, values) of the CTA's
// contiguous row range through an S-stage shared-memory ring with bulk copies and
// keeps a sliding window of x rows (ring of WCAP rows) ahead of the rows in flight;
// T consumer threads turn each stage into products (entry-parallel: P[i] = v * x[col])
// and, per sub-block of T rows, one thread per row adds its products in entry order.
struct S2Args {
    const int* rp;
    const uint32_t* ci;
    const double* v;
    const double* x;
    double* y;
    int n, band, rows_per_cta, wcap;
    int pf_entries;          // L2 prefetch distance of the producer (entries; 0 = off)
};
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ void bar_consumers(int nthreads) {
    asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

template <int M, int T, int SE, int S, int PCAP>
__global__ void __launch_bounds__(T + 32, 1) k_stream2(S2Args a) {
    static_assert(PCAP % SE == 0, "a product piece is a whole number of stages");
    extern __shared__ __align__(128) unsigned char sm[];
    const int WCAP = a.wcap;
    double* xs = reinterpret_cast<double*>(sm);                              // WCAP x M
    double* P = xs + (size_t)WCAP * M;                                       // PCAP x M
    unsigned char* ring = reinterpret_cast<unsigned char*>(P + (size_t)PCAP * M);   // S x (SE*4 + SE*8)
    constexpr int STB = SE * 12;
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + S * STB);
    uint64_t* empty = full + S;
    int* slot_rb = reinterpret_cast<int*>(empty + S);                        // producer-private
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) { mb_init(full + s, 1); mb_init(empty + s, T / 32); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int R0 = min(a.n, (int)blockIdx.x * a.rows_per_cta);
    const int R1 = min(a.n, R0 + a.rows_per_cta);
    if (R0 >= R1) return;
    const int nsb = (R1 - R0 + T - 1) / T;
    if (threadIdx.x >= T) {
        // ---------------- producer warp
        const int lane = threadIdx.x - T;
        int issued = 0, released = 0;
        int pf_e = __ldg(a.rp + R0) & ~3;              // entries below pf_e are prefetched into L2
        const int e_end = __ldg(a.rp + R1);
        int whi = max(0, R0 - a.band);                 // x rows [.., whi) are loaded (or being loaded)
        if (M == 1) whi &= ~1;
        for (int sb0 = 0; sb0 < nsb; sb0 += 32) {
            const int rbj = min(R1, R0 + (sb0 + lane) * T);
            const int ebj = __ldg(a.rp + rbj);
            int eej = __shfl_down_sync(~0u, ebj, 1);
            if (lane == 31) eej = __ldg(a.rp + min(R1, rbj + T));
            const int cntj = min(32, nsb - sb0);
            for (int j = 0; j < cntj; ++j) {
                const int eb = __shfl_sync(~0u, ebj, j), ee = __shfl_sync(~0u, eej, j);
                if (lane != 0) continue;
                const int rb = R0 + (sb0 + j) * T, re = min(R1, rb + T);
                const int a0 = eb & ~3;
                bool first = true;
                for (int cs = a0; cs < ee; cs += SE, first = false) {
                    const int slot = issued % S;
                    while (released < issued - S + 1) {
                        mb_wait(empty + released % S, (released / S) & 1);
                        ++released;
                    }
                    const int len = min(SE, (ee - cs + 3) & ~3);
                    if (a.pf_entries) {
                        const int tgt = min(e_end, cs + a.pf_entries);
                        while (pf_e < tgt) {
                            const int pl = min(2048, (e_end - pf_e + 3) & ~3);
                            prefetch_l2(a.ci + pf_e, (uint32_t)pl * 4);
                            prefetch_l2(a.v + pf_e, (uint32_t)pl * 8);
                            pf_e += pl;
                        }
                    }
                    uint32_t tx = (uint32_t)len * 12;
                    int wnew = whi;
                    if (first) {
                        wnew = min(a.n, re + a.band);
                        if (M == 1) wnew = min(a.n, (wnew + 1) & ~1);
                        if (wnew > whi) {
                            // rows below wnew - WCAP are overwritten: every stage still in
                            // flight must belong to a sub-block starting at or above that + band
                            while (released < issued && wnew - WCAP > slot_rb[released % S] - a.band) {
                                mb_wait(empty + released % S, (released / S) & 1);
                                ++released;
                            }
                            tx += (uint32_t)(wnew - whi) * M * 8;
                        } else wnew = whi;
                    }
                    slot_rb[slot] = rb;
                    mb_expect(full + slot, tx);
                    unsigned char* st = ring + slot * STB;
                    bulk_g2s(st, a.ci + cs, (uint32_t)len * 4, full + slot);
                    bulk_g2s(st + SE * 4, a.v + cs, (uint32_t)len * 8, full + slot);
                    if (wnew > whi) {
                        int c = whi;
                        while (c < wnew) {             // split at the ring wrap and at 32 KB
                            const int sl = c % WCAP;
                            const int cnt = min(min(wnew - c, WCAP - sl), 32768 / (M * 8));
                            bulk_g2s(xs + (size_t)sl * M, a.x + (size_t)c * M, (uint32_t)cnt * M * 8, full + slot);
                            c += cnt;
                        }
                        whi = wnew;
                    }
                    ++issued;
                }
            }
        }
        return;
    }
    // ---------------- consumers
    const int warp = threadIdx.x / 32;
    int it = 0;                                        // stage counter (same sequence as the producer)
    for (int sb = 0; sb < nsb; ++sb) {
        const int rb = R0 + sb * T, re = min(R1, rb + T);
        const int row = rb + threadIdx.x;
        const int eb = __ldg(a.rp + rb), ee = __ldg(a.rp + re);
        int lo = 0, hi = 0;
        if (row < re) { lo = __ldg(a.rp + row); hi = __ldg(a.rp + row + 1); }
        const int wbase = max(0, rb - a.band) & ~1;    // lowest x row this sub-block may read
        const int wslot = wbase % WCAP;
        double acc[M];
#pragma unroll
        for (int i = 0; i < M; ++i) acc[i] = 0.0;
        const int a0 = eb & ~3;
        for (int pb = a0; pb < ee; pb += PCAP) {       // product pieces (usually one per sub-block)
            const int pe = min(ee, pb + PCAP);
            for (int cs = pb; cs < pe; cs += SE, ++it) {
                const int slot = it % S;
                mb_wait(full + slot, (it / S) & 1);
                const uint32_t* sc = reinterpret_cast<const uint32_t*>(ring + slot * STB);
                const double* sv = reinterpret_cast<const double*>(ring + slot * STB + SE * 4);
                const int i0 = max(eb, cs) - cs, i1 = min(pe, cs + SE) - cs;
                constexpr int U1 = 4;
                for (int ib = i0 + threadIdx.x; ib < i1; ib += T * U1) {
                    int sl[U1]; double v[U1];
#pragma unroll
                    for (int u = 0; u < U1; ++u) {
                        const int i = min(ib + u * T, i1 - 1);
                        sl[u] = wslot + ((int)sc[i] - wbase);
                        v[u] = sv[i];
                    }
                    fence();
                    double px[U1][M];
#pragma unroll
                    for (int u = 0; u < U1; ++u) {
                        if (sl[u] >= WCAP) sl[u] -= WCAP;
                        if constexpr (M == 1) px[u][0] = xs[sl[u]];
                        else {
                            const double2 t = *reinterpret_cast<const double2*>(xs + 2 * sl[u]);
                            px[u][0] = t.x; px[u][1] = t.y;
                        }
                    }
                    fence();
#pragma unroll
                    for (int u = 0; u < U1; ++u) {
                        const int i = ib + u * T;
                        if (i < i1) {
                            if constexpr (M == 1) P[cs - pb + i] = mul(v[u], px[u][0]);
                            else *reinterpret_cast<double2*>(P + 2 * (cs - pb + i)) =
                                     make_double2(mul(v[u], px[u][0]), mul(v[u], px[u][1]));
                        }
                    }
                }
                __syncwarp();
                if (threadIdx.x % 32 == 0) mb_arrive(empty + slot);
            }
            bar_consumers(T);
            const int klo = max(lo, pb) - pb, khi = min(hi, pe) - pb;
            constexpr int U2 = 4;
            for (int k = klo; k < khi; k += U2) {
                double t[U2][M];
#pragma unroll
                for (int u = 0; u < U2; ++u) {
                    const int kk = min(k + u, khi - 1);
                    if constexpr (M == 1) t[u][0] = P[kk];
                    else {
                        const double2 q = *reinterpret_cast<const double2*>(P + 2 * kk);
                        t[u][0] = q.x; t[u][1] = q.y;
                    }
                }
                fence();
#pragma unroll
                for (int u = 0; u < U2; ++u)
                    if (k + u < khi)
#pragma unroll
                        for (int i = 0; i < M; ++i) acc[i] = add(acc[i], t[u][i]);
            }
            bar_consumers(T);
        }
        if (row < re) {
            if constexpr (M == 1) a.y[row] = acc[0];
            else *reinterpret_cast<double2*>(a.y + 2 * (size_t)row) = make_double2(acc[0], acc[1]);
        }
        (void)warp;
    }
}

template <int M, int T, int SE, int S, int PCAP>
__global__ void __launch_bounds__(T + 32, 1) k_stream4(S2Args a) {
    static_assert(PCAP % SE == 0, "a product piece is a whole number of stages");
    extern __shared__ __align__(128) unsigned char sm[];
    const int WCAP = a.wcap;
    double* xs = reinterpret_cast<double*>(sm);                              // WCAP x M
    double* P = xs + (size_t)WCAP * M;                                       // PCAP x M
    unsigned char* ring = reinterpret_cast<unsigned char*>(P + (size_t)PCAP * M);   // S x (SE*4 + SE*8)
    constexpr int STB = SE * 12;
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + S * STB);
    uint64_t* empty = full + S;
    int* slot_rb = reinterpret_cast<int*>(empty + S);                        // producer-private
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) { mb_init(full + s, 1); mb_init(empty + s, T / 32); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int R0 = min(a.n, (int)blockIdx.x * a.rows_per_cta);
    const int R1 = min(a.n, R0 + a.rows_per_cta);
    if (R0 >= R1) return;
    const int nsb = (R1 - R0 + T - 1) / T;
    if (threadIdx.x >= T) {
        // ---------------- producer warp
        const int lane = threadIdx.x - T;
        int issued = 0, released = 0;
        int pf_e = __ldg(a.rp + R0) & ~3;              // entries below pf_e are prefetched into L2
        const int e_end = __ldg(a.rp + R1);
        int whi = max(0, R0 - a.band);                 // x rows [.., whi) are loaded (or being loaded)
        if (M == 1) whi &= ~1;
        for (int sb0 = 0; sb0 < nsb; sb0 += 32) {
            const int rbj = min(R1, R0 + (sb0 + lane) * T);
            const int ebj = __ldg(a.rp + rbj);
            int eej = __shfl_down_sync(~0u, ebj, 1);
            if (lane == 31) eej = __ldg(a.rp + min(R1, rbj + T));
            const int cntj = min(32, nsb - sb0);
            for (int j = 0; j < cntj; ++j) {
                const int eb = __shfl_sync(~0u, ebj, j), ee = __shfl_sync(~0u, eej, j);
                if (lane != 0) continue;
                const int rb = R0 + (sb0 + j) * T, re = min(R1, rb + T);
                const int a0 = eb & ~3;
                bool first = true;
                for (int cs = a0; cs < ee; cs += SE, first = false) {
                    const int slot = issued % S;
                    while (released < issued - S + 1) {
                        mb_wait(empty + released % S, (released / S) & 1);
                        ++released;
                    }
                    const int len = min(SE, (ee - cs + 3) & ~3);
                    if (a.pf_entries > 0) {
                        const int tgt = min(e_end, cs + a.pf_entries);
                        while (pf_e < tgt) {
                            const int pl = min(2048, (e_end - pf_e + 3) & ~3);
                            prefetch_l2(a.ci + pf_e, (uint32_t)pl * 4);
                            prefetch_l2(a.v + pf_e, (uint32_t)pl * 8);
                            pf_e += pl;
                        }
                    }
                    uint32_t tx = (uint32_t)len * 12;
                    int wnew = whi;
                    if (first) {
                        wnew = min(a.n, re + a.band);
                        if (M == 1) wnew = min(a.n, (wnew + 1) & ~1);
                        if (wnew > whi) {
                            // rows below wnew - WCAP are overwritten: every stage still in
                            // flight must belong to a sub-block starting at or above that + band
                            while (released < issued && wnew - WCAP > slot_rb[released % S] - a.band) {
                                mb_wait(empty + released % S, (released / S) & 1);
                                ++released;
                            }
                            tx += (uint32_t)(wnew - whi) * M * 8;
                        } else wnew = whi;
                    }
                    slot_rb[slot] = rb;
                    mb_expect(full + slot, tx);
                    unsigned char* st = ring + slot * STB;
                    bulk_g2s(st, a.ci + cs, (uint32_t)len * 4, full + slot);
                    bulk_g2s(st + SE * 4, a.v + cs, (uint32_t)len * 8, full + slot);
                    if (wnew > whi) {
                        int c = whi;
                        while (c < wnew) {             // split at the ring wrap and at 32 KB
                            const int sl = c % WCAP;
                            const int cnt = min(min(wnew - c, WCAP - sl), 32768 / (M * 8));
                            bulk_g2s(xs + (size_t)sl * M, a.x + (size_t)c * M, (uint32_t)cnt * M * 8, full + slot);
                            c += cnt;
                        }
                        whi = wnew;
                    }
                    ++issued;
                }
            }
        }
        return;
    }
    // ---------------- consumers
    const int warp = threadIdx.x / 32;
    int it = 0;                                        // stage counter (same sequence as the producer)
    // row pointers of the NEXT sub-block are loaded while this one is processed
    int n_eb = __ldg(a.rp + R0), n_ee = __ldg(a.rp + min(R1, R0 + T));
    int n_lo = __ldg(a.rp + min(R1, R0 + (int)threadIdx.x)), n_hi = __ldg(a.rp + min(R1, R0 + (int)threadIdx.x + 1));
    for (int sb = 0; sb < nsb; ++sb) {
        const int rb = R0 + sb * T, re = min(R1, rb + T);
        const int row = rb + threadIdx.x;
        const int eb = n_eb, ee = n_ee;
        const int lo = n_lo, hi = n_hi;                // (rows past the range: lo == hi)
        {
            const int nb = min(R1, rb + T), ne = min(R1, rb + 2 * T);
            n_eb = ee;
            n_ee = __ldg(a.rp + ne);
            n_lo = __ldg(a.rp + min(R1, nb + (int)threadIdx.x));
            n_hi = __ldg(a.rp + min(R1, nb + (int)threadIdx.x + 1));
        }
        const int wbase = max(0, rb - a.band) & ~1;    // lowest x row this sub-block may read
        const int wslot = wbase % WCAP;
        double acc[M];
#pragma unroll
        for (int i = 0; i < M; ++i) acc[i] = 0.0;
        const int a0 = eb & ~3;
        for (int pb = a0; pb < ee; pb += PCAP) {       // product pieces (usually one per sub-block)
            const int pe = min(ee, pb + PCAP);
            for (int cs = pb; cs < pe; cs += SE, ++it) {
                const int slot = it % S;
                mb_wait(full + slot, (it / S) & 1);
                const uint32_t* sc = reinterpret_cast<const uint32_t*>(ring + slot * STB);
                const double* sv = reinterpret_cast<const double*>(ring + slot * STB + SE * 4);
                const int i0 = max(eb, cs) - cs, i1 = min(pe, cs + SE) - cs;
                constexpr int U1 = 4;
                if (a.pf_entries != -1)
                for (int ib = i0 + threadIdx.x; ib < i1; ib += T * U1) {
                    int sl[U1]; double v[U1];
#pragma unroll
                    for (int u = 0; u < U1; ++u) {
                        const int i = min(ib + u * T, i1 - 1);
                        sl[u] = wslot + ((int)sc[i] - wbase);
                        v[u] = sv[i];
                    }
                    fence();
                    double px[U1][M];
#pragma unroll
                    for (int u = 0; u < U1; ++u) {
                        if (sl[u] >= WCAP) sl[u] -= WCAP;
                        if constexpr (M == 1) px[u][0] = xs[sl[u]];
                        else {
                            const double2 t = *reinterpret_cast<const double2*>(xs + 2 * sl[u]);
                            px[u][0] = t.x; px[u][1] = t.y;
                        }
                    }
                    fence();
#pragma unroll
                    for (int u = 0; u < U1; ++u) {
                        const int i = ib + u * T;
                        if (i < i1) {
                            if constexpr (M == 1) P[cs - pb + i] = mul(v[u], px[u][0]);
                            else *reinterpret_cast<double2*>(P + 2 * (cs - pb + i)) =
                                     make_double2(mul(v[u], px[u][0]), mul(v[u], px[u][1]));
                        }
                    }
                }
                __syncwarp();
                if (threadIdx.x % 32 == 0) mb_arrive(empty + slot);
            }
            bar_consumers(T);
            const int klo = max(lo, pb) - pb, khi = min(hi, pe) - pb;
            constexpr int U2 = 4;
            if (a.pf_entries != -1 && a.pf_entries != -2)
            for (int k = klo; k < khi; k += U2) {
                double t[U2][M];
#pragma unroll
                for (int u = 0; u < U2; ++u) {
                    const int kk = min(k + u, khi - 1);
                    if constexpr (M == 1) t[u][0] = P[kk];
                    else {
                        const double2 q = *reinterpret_cast<const double2*>(P + 2 * kk);
                        t[u][0] = q.x; t[u][1] = q.y;
                    }
                }
                fence();
#pragma unroll
                for (int u = 0; u < U2; ++u)
                    if (k + u < khi)
#pragma unroll
                        for (int i = 0; i < M; ++i) acc[i] = add(acc[i], t[u][i]);
            }
            bar_consumers(T);
        }
        if (row < re) {
            if constexpr (M == 1) a.y[row] = acc[0];
            else *reinterpret_cast<double2*>(a.y + 2 * (size_t)row) = make_double2(acc[0], acc[1]);
        }
        (void)warp;
    }
}

template <int M, int T, int SE, int S, int PCAP>
__global__ void __launch_bounds__(T + 32, 1) k_stream5(S2Args a) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int WCAP = a.wcap;
    double* xs = reinterpret_cast<double*>(sm);                              // WCAP x M
    double* P = xs + (size_t)WCAP * M;                                       // PCAP x M
    unsigned char* ring = reinterpret_cast<unsigned char*>(P + (size_t)PCAP * M * 2);   // (P: two buffers)   // S x (SE*4 + SE*8)
    constexpr int STB = SE * 12;
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + S * STB);
    uint64_t* empty = full + S;
    int* slot_rb = reinterpret_cast<int*>(empty + S);                        // producer-private
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) { mb_init(full + s, 1); mb_init(empty + s, T / 32); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int R0 = min(a.n, (int)blockIdx.x * a.rows_per_cta);
    const int R1 = min(a.n, R0 + a.rows_per_cta);
    if (R0 >= R1) return;
    const int nsb = (R1 - R0 + T - 1) / T;
    if (threadIdx.x >= T) {
        // ---------------- producer warp
        const int lane = threadIdx.x - T;
        int issued = 0, released = 0;
        int pf_e = __ldg(a.rp + R0) & ~3;              // entries below pf_e are prefetched into L2
        const int e_end = __ldg(a.rp + R1);
        int whi = max(0, R0 - a.band);                 // x rows [.., whi) are loaded (or being loaded)
        if (M == 1) whi &= ~1;
        for (int sb0 = 0; sb0 < nsb; sb0 += 32) {
            const int rbj = min(R1, R0 + (sb0 + lane) * T);
            const int ebj = __ldg(a.rp + rbj);
            int eej = __shfl_down_sync(~0u, ebj, 1);
            if (lane == 31) eej = __ldg(a.rp + min(R1, rbj + T));
            const int cntj = min(32, nsb - sb0);
            for (int j = 0; j < cntj; ++j) {
                const int eb = __shfl_sync(~0u, ebj, j), ee = __shfl_sync(~0u, eej, j);
                if (lane != 0) continue;
                const int rb = R0 + (sb0 + j) * T, re = min(R1, rb + T);
                const int a0 = eb & ~3;
                bool first = true;
                for (int cs = a0; cs < ee; cs += SE, first = false) {
                    const int slot = issued % S;
                    while (released < issued - S + 1) {
                        mb_wait(empty + released % S, (released / S) & 1);
                        ++released;
                    }
                    const int len = min(SE, (ee - cs + 3) & ~3);
                    if (a.pf_entries > 0) {
                        const int tgt = min(e_end, cs + a.pf_entries);
                        while (pf_e < tgt) {
                            const int pl = min(2048, (e_end - pf_e + 3) & ~3);
                            prefetch_l2(a.ci + pf_e, (uint32_t)pl * 4);
                            prefetch_l2(a.v + pf_e, (uint32_t)pl * 8);
                            pf_e += pl;
                        }
                    }
                    uint32_t tx = (uint32_t)len * 12;
                    int wnew = whi;
                    if (first) {
                        wnew = min(a.n, re + a.band);
                        if (M == 1) wnew = min(a.n, (wnew + 1) & ~1);
                        if (wnew > whi) {
                            // rows below wnew - WCAP are overwritten: every stage still in
                            // flight must belong to a sub-block starting at or above that + band
                            while (released < issued && wnew - WCAP > slot_rb[released % S] - a.band) {
                                mb_wait(empty + released % S, (released / S) & 1);
                                ++released;
                            }
                            tx += (uint32_t)(wnew - whi) * M * 8;
                        } else wnew = whi;
                    }
                    slot_rb[slot] = rb;
                    mb_expect(full + slot, tx);
                    unsigned char* st = ring + slot * STB;
                    bulk_g2s(st, a.ci + cs, (uint32_t)len * 4, full + slot);
                    bulk_g2s(st + SE * 4, a.v + cs, (uint32_t)len * 8, full + slot);
                    if (wnew > whi) {
                        int c = whi;
                        while (c < wnew) {             // split at the ring wrap and at 32 KB
                            const int sl = c % WCAP;
                            const int cnt = min(min(wnew - c, WCAP - sl), 32768 / (M * 8));
                            bulk_g2s(xs + (size_t)sl * M, a.x + (size_t)c * M, (uint32_t)cnt * M * 8, full + slot);
                            c += cnt;
                        }
                        whi = wnew;
                    }
                    ++issued;
                }
            }
        }
        return;
    }
    // ---------------- consumers: step s = products of sub-block s (into P[s & 1]) fused with
    // the ordered row sums of sub-block s - 1 (from P[(s - 1) & 1]); one barrier per step.
    // Requires every sub-block's entries (+ 3 of alignment) to fit PCAP (checked on the host).
    int it = 0;
    int n_eb = __ldg(a.rp + R0), n_ee = __ldg(a.rp + min(R1, R0 + T));
    int n_lo = __ldg(a.rp + min(R1, R0 + (int)threadIdx.x)), n_hi = __ldg(a.rp + min(R1, R0 + (int)threadIdx.x + 1));
    int p2_a0 = 0, p2_lo = 0, p2_hi = 0, p2_row = -1;
    for (int s = 0; s <= nsb; ++s) {
        const int rb = R0 + s * T, re = min(R1, rb + T);
        int eb = n_eb, ee = n_ee;
        const int lo = n_lo, hi = n_hi;
        if (s >= nsb) ee = eb;
        {
            const int nb = min(R1, rb + T), ne = min(R1, rb + 2 * T);
            n_eb = n_ee;
            n_ee = __ldg(a.rp + ne);
            n_lo = __ldg(a.rp + min(R1, nb + (int)threadIdx.x));
            n_hi = __ldg(a.rp + min(R1, nb + (int)threadIdx.x + 1));
        }
        const int a0 = eb & ~3;
        double* P1 = P + (size_t)(s & 1) * PCAP * M;
        const double* P2 = P + (size_t)((s & 1) ^ 1) * PCAP * M;
        const int wbase = max(0, rb - a.band) & ~1;
        const int wslot = wbase % WCAP;
        int k2 = p2_lo - p2_a0;
        const int k2e = p2_hi - p2_a0;
        double acc[M];
#pragma unroll
        for (int i = 0; i < M; ++i) acc[i] = 0.0;
        constexpr int U1 = 4, U2 = 4;
        auto sum_batch = [&]() {           // U2 products of the previous sub-block's row, in order
            double t[U2][M];
#pragma unroll
            for (int u = 0; u < U2; ++u) {
                const int kk = max(0, min(k2 + u, k2e - 1));
                if constexpr (M == 1) t[u][0] = P2[kk];
                else {
                    const double2 q = *reinterpret_cast<const double2*>(P2 + 2 * kk);
                    t[u][0] = q.x; t[u][1] = q.y;
                }
            }
#pragma unroll
            for (int u = 0; u < U2; ++u) {
                const bool on = k2 + u < k2e;
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    const double r = add(acc[i], t[u][i]);
                    acc[i] = on ? r : acc[i];
                }
            }
            k2 += U2;
        };
        for (int cs = a0; s < nsb && cs < ee; cs += SE, ++it) {
            const int slot = it % S;
            mb_wait(full + slot, (it / S) & 1);
            const uint32_t* sc = reinterpret_cast<const uint32_t*>(ring + slot * STB);
            const double* sv = reinterpret_cast<const double*>(ring + slot * STB + SE * 4);
            const int i0 = max(eb, cs) - cs, i1 = min(ee, cs + SE) - cs;
            for (int ib = i0 + threadIdx.x; ib < i1; ib += T * U1) {
                int sl[U1]; double v[U1];
#pragma unroll
                for (int u = 0; u < U1; ++u) {
                    const int i = min(ib + u * T, i1 - 1);
                    sl[u] = wslot + ((int)sc[i] - wbase);
                    v[u] = sv[i];
                }
                double px[U1][M];
#pragma unroll
                for (int u = 0; u < U1; ++u) {
                    if (sl[u] >= WCAP) sl[u] -= WCAP;
                    if constexpr (M == 1) px[u][0] = xs[sl[u]];
                    else {
                        const double2 t = *reinterpret_cast<const double2*>(xs + 2 * sl[u]);
                        px[u][0] = t.x; px[u][1] = t.y;
                    }
                }
                sum_batch();
#pragma unroll
                for (int u = 0; u < U1; ++u) {
                    const int i = ib + u * T;
                    if (i < i1) {
                        if constexpr (M == 1) P1[cs - a0 + i] = mul(v[u], px[u][0]);
                        else *reinterpret_cast<double2*>(P1 + 2 * (cs - a0 + i)) =
                                 make_double2(mul(v[u], px[u][0]), mul(v[u], px[u][1]));
                    }
                }
            }
            __syncwarp();
            if (threadIdx.x % 32 == 0) mb_arrive(empty + slot);
        }
        while (k2 < k2e) sum_batch();
        if (p2_row >= 0) {
            if constexpr (M == 1) a.y[p2_row] = acc[0];
            else *reinterpret_cast<double2*>(a.y + 2 * (size_t)p2_row) = make_double2(acc[0], acc[1]);
        }
        bar_consumers(T);
        p2_a0 = a0; p2_lo = lo; p2_hi = hi;
        p2_row = (s < nsb && rb + (int)threadIdx.x < re) ? rb + (int)threadIdx.x : -1;
    }
}

// stream6: warp-specialised consumers: NP product threads turn stages into products
// (P[s & 1]) while T sum threads (one per row) add the previous sub-block's products in
// entry order; P buffers are handed over with mbarriers (pfull / pempty).
template <int M, int T, int NP, int SE, int S, int PCAP>
__global__ void __launch_bounds__(T + NP + 32, 1) k_stream6(S2Args a) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int WCAP = a.wcap;
    double* xs = reinterpret_cast<double*>(sm);                              // WCAP x M
    double* P = xs + (size_t)WCAP * M;                                       // PCAP x M
    unsigned char* ring = reinterpret_cast<unsigned char*>(P + (size_t)PCAP * M * 2);   // (P: two buffers)   // S x (SE*4 + SE*8)
    constexpr int STB = SE * 12;
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + S * STB);
    uint64_t* empty = full + S;
    uint64_t* pfull = empty + S;                                             // [2]
    uint64_t* pempty = pfull + 2;                                            // [2]
    int* slot_rb = reinterpret_cast<int*>(pempty + 2);                       // producer-private
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) { mb_init(full + s, 1); mb_init(empty + s, NP / 32); }
        for (int s = 0; s < 2; ++s) { mb_init(pfull + s, NP / 32); mb_init(pempty + s, T / 32); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int R0 = min(a.n, (int)blockIdx.x * a.rows_per_cta);
    const int R1 = min(a.n, R0 + a.rows_per_cta);
    if (R0 >= R1) return;
    const int nsb = (R1 - R0 + T - 1) / T;
    if (threadIdx.x >= T + NP) {
        // ---------------- producer warp
        const int lane = threadIdx.x - T - NP;
        int issued = 0, released = 0;
        int pf_e = __ldg(a.rp + R0) & ~3;              // entries below pf_e are prefetched into L2
        const int e_end = __ldg(a.rp + R1);
        int whi = max(0, R0 - a.band);                 // x rows [.., whi) are loaded (or being loaded)
        if (M == 1) whi &= ~1;
        for (int sb0 = 0; sb0 < nsb; sb0 += 32) {
            const int rbj = min(R1, R0 + (sb0 + lane) * T);
            const int ebj = __ldg(a.rp + rbj);
            int eej = __shfl_down_sync(~0u, ebj, 1);
            if (lane == 31) eej = __ldg(a.rp + min(R1, rbj + T));
            const int cntj = min(32, nsb - sb0);
            for (int j = 0; j < cntj; ++j) {
                const int eb = __shfl_sync(~0u, ebj, j), ee = __shfl_sync(~0u, eej, j);
                if (lane != 0) continue;
                const int rb = R0 + (sb0 + j) * T, re = min(R1, rb + T);
                const int a0 = eb & ~3;
                bool first = true;
                for (int cs = a0; cs < ee; cs += SE, first = false) {
                    const int slot = issued % S;
                    while (released < issued - S + 1) {
                        mb_wait(empty + released % S, (released / S) & 1);
                        ++released;
                    }
                    const int len = min(SE, (ee - cs + 3) & ~3);
                    if (a.pf_entries > 0) {
                        const int tgt = min(e_end, cs + a.pf_entries);
                        while (pf_e < tgt) {
                            const int pl = min(2048, (e_end - pf_e + 3) & ~3);
                            prefetch_l2(a.ci + pf_e, (uint32_t)pl * 4);
                            prefetch_l2(a.v + pf_e, (uint32_t)pl * 8);
                            pf_e += pl;
                        }
                    }
                    uint32_t tx = (uint32_t)len * 12;
                    int wnew = whi;
                    if (first) {
                        wnew = min(a.n, re + a.band);
                        if (M == 1) wnew = min(a.n, (wnew + 1) & ~1);
                        if (wnew > whi) {
                            // rows below wnew - WCAP are overwritten: every stage still in
                            // flight must belong to a sub-block starting at or above that + band
                            while (released < issued && wnew - WCAP > slot_rb[released % S] - a.band) {
                                mb_wait(empty + released % S, (released / S) & 1);
                                ++released;
                            }
                            tx += (uint32_t)(wnew - whi) * M * 8;
                        } else wnew = whi;
                    }
                    slot_rb[slot] = rb;
                    mb_expect(full + slot, tx);
                    unsigned char* st = ring + slot * STB;
                    bulk_g2s(st, a.ci + cs, (uint32_t)len * 4, full + slot);
                    bulk_g2s(st + SE * 4, a.v + cs, (uint32_t)len * 8, full + slot);
                    if (wnew > whi) {
                        int c = whi;
                        while (c < wnew) {             // split at the ring wrap and at 32 KB
                            const int sl = c % WCAP;
                            const int cnt = min(min(wnew - c, WCAP - sl), 32768 / (M * 8));
                            bulk_g2s(xs + (size_t)sl * M, a.x + (size_t)c * M, (uint32_t)cnt * M * 8, full + slot);
                            c += cnt;
                        }
                        whi = wnew;
                    }
                    ++issued;
                }
            }
        }
        return;
    }
    if (threadIdx.x >= T) {
        // ---------------- product warps
        const int pt = threadIdx.x - T;
        int it = 0;
        int n_eb = __ldg(a.rp + R0), n_ee = __ldg(a.rp + min(R1, R0 + T));
        for (int s = 0; s < nsb; ++s) {
            const int rb = R0 + s * T;
            const int eb = n_eb, ee = n_ee;
            n_eb = n_ee;
            n_ee = __ldg(a.rp + min(R1, rb + 2 * T));
            const int a0 = eb & ~3;
            double* P1 = P + (size_t)(s & 1) * PCAP * M;
            const int wbase = max(0, rb - a.band) & ~1;
            const int wslot = wbase % WCAP;
            if (s >= 2) mb_wait(pempty + (s & 1), ((s >> 1) - 1) & 1);     // sums of sub-block s - 2 done
            constexpr int U1 = (SE + NP - 1) / NP < 4 ? (SE + NP - 1) / NP : 4;
            for (int cs = a0; cs < ee; cs += SE, ++it) {
                const int slot = it % S;
                mb_wait(full + slot, (it / S) & 1);
                const uint32_t* sc = reinterpret_cast<const uint32_t*>(ring + slot * STB);
                const double* sv = reinterpret_cast<const double*>(ring + slot * STB + SE * 4);
                const int i0 = max(eb, cs) - cs, i1 = min(ee, cs + SE) - cs;
                for (int ib = i0 + pt; ib < i1; ib += NP * U1) {
                    int sl[U1]; double v[U1];
#pragma unroll
                    for (int u = 0; u < U1; ++u) {
                        const int i = min(ib + u * NP, i1 - 1);
                        sl[u] = wslot + ((int)sc[i] - wbase);
                        v[u] = sv[i];
                    }
                    fence();
                    double px[U1][M];
#pragma unroll
                    for (int u = 0; u < U1; ++u) {
                        if (sl[u] >= WCAP) sl[u] -= WCAP;
                        if constexpr (M == 1) px[u][0] = xs[sl[u]];
                        else {
                            const double2 t = *reinterpret_cast<const double2*>(xs + 2 * sl[u]);
                            px[u][0] = t.x; px[u][1] = t.y;
                        }
                    }
                    fence();
#pragma unroll
                    for (int u = 0; u < U1; ++u) {
                        const int i = ib + u * NP;
                        if (i < i1) {
                            if constexpr (M == 1) P1[cs - a0 + i] = mul(v[u], px[u][0]);
                            else *reinterpret_cast<double2*>(P1 + 2 * (cs - a0 + i)) =
                                     make_double2(mul(v[u], px[u][0]), mul(v[u], px[u][1]));
                        }
                    }
                }
                __syncwarp();
                if (threadIdx.x % 32 == 0) mb_arrive(empty + slot);
            }
            __syncwarp();
            if (threadIdx.x % 32 == 0) mb_arrive(pfull + (s & 1));
        }
        return;
    }
    // ---------------- sum warps: one thread per row of the sub-block
    int n_lo = __ldg(a.rp + min(R1, R0 + (int)threadIdx.x)), n_hi = __ldg(a.rp + min(R1, R0 + (int)threadIdx.x + 1));
    int n_eb = __ldg(a.rp + R0);
    for (int s = 0; s < nsb; ++s) {
        const int rb = R0 + s * T, re = min(R1, rb + T);
        const int row = rb + threadIdx.x;
        const int lo = n_lo, hi = n_hi, a0 = n_eb & ~3;
        {
            const int nb = min(R1, rb + T);
            n_eb = __ldg(a.rp + nb);
            n_lo = __ldg(a.rp + min(R1, nb + (int)threadIdx.x));
            n_hi = __ldg(a.rp + min(R1, nb + (int)threadIdx.x + 1));
        }
        const double* P2 = P + (size_t)(s & 1) * PCAP * M;
        mb_wait(pfull + (s & 1), (s >> 1) & 1);
        double acc[M];
#pragma unroll
        for (int i = 0; i < M; ++i) acc[i] = 0.0;
        constexpr int U2 = 4;
        const int klo = lo - a0, khi = hi - a0;
        for (int k = klo; k < khi; k += U2) {
            double t[U2][M];
#pragma unroll
            for (int u = 0; u < U2; ++u) {
                const int kk = min(k + u, khi - 1);
                if constexpr (M == 1) t[u][0] = P2[kk];
                else {
                    const double2 q = *reinterpret_cast<const double2*>(P2 + 2 * kk);
                    t[u][0] = q.x; t[u][1] = q.y;
                }
            }
            fence();
#pragma unroll
            for (int u = 0; u < U2; ++u)
                if (k + u < khi)
#pragma unroll
                    for (int i = 0; i < M; ++i) acc[i] = add(acc[i], t[u][i]);
        }
        __syncwarp();
        if (threadIdx.x % 32 == 0) mb_arrive(pempty + (s & 1));
        if (row < re) {
            if constexpr (M == 1) a.y[row] = acc[0];
            else *reinterpret_cast<double2*>(a.y + 2 * (size_t)row) = make_double2(acc[0], acc[1]);
        }
    }
}

// stream3: NT consumer teams of TT threads; team q owns sub-blocks q, q + NT, ... (TT rows
// each) and its own product buffer, so one team's ordered row sums overlap the other's
// products; product i sits at P[i + i/16] (row starts ~16 apart fall into different banks).
__device__ __forceinline__ void bar_team(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ int ppos(int i) { return i + (i >> 4); }
template <int M, int TT, int NT, int SE, int S, int PCAP>
__global__ void __launch_bounds__(TT * NT + 32, 1) k_stream3(S2Args a) {
    // S = ring slots PER TEAM: a team only ever waits on slots whose previous use it
    // consumed itself (mbarrier parity waits alias two phases apart)
    constexpr int T = TT * NT;
    constexpr int NS = S * NT;
    constexpr int PSZ = PCAP + PCAP / 16 + 2;
    static_assert(PCAP % SE == 0, "a product piece is a whole number of stages");
    extern __shared__ __align__(128) unsigned char sm[];
    const int WCAP = a.wcap;
    double* xs = reinterpret_cast<double*>(sm);                              // WCAP x M
    double* P = xs + (size_t)WCAP * M;                                       // NT x PSZ x M
    unsigned char* ring = reinterpret_cast<unsigned char*>(P + (size_t)PSZ * M * NT);   // NS x (SE*4 + SE*8)
    constexpr int STB = SE * 12;
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + NS * STB);
    uint64_t* empty = full + NS;
    int* slot_rb = reinterpret_cast<int*>(empty + NS);                       // producer-private
    int* iss = slot_rb + NS;                                                 // stages issued / released per team
    int* rel = iss + NT;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) { mb_init(full + s, 1); mb_init(empty + s, TT / 32); }
        for (int q = 0; q < NT; ++q) { iss[q] = 0; rel[q] = 0; }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int R0 = min(a.n, (int)blockIdx.x * a.rows_per_cta);
    const int R1 = min(a.n, R0 + a.rows_per_cta);
    if (R0 >= R1) return;
    const int nsb = (R1 - R0 + TT - 1) / TT;
    if (threadIdx.x >= T) {
        // ---------------- producer warp
        const int lane = threadIdx.x - T;
        int whi = max(0, R0 - a.band);                 // x rows [.., whi) are loaded (or being loaded)
        if (M == 1) whi &= ~1;
        auto release_one = [&](int q) {
            const int r = rel[q];
            mb_wait(empty + q * S + r % S, (r / S) & 1);
            rel[q] = r + 1;
        };
        for (int sb0 = 0; sb0 < nsb; sb0 += 32) {
            const int rbj = min(R1, R0 + (sb0 + lane) * TT);
            const int ebj = __ldg(a.rp + rbj);
            int eej = __shfl_down_sync(~0u, ebj, 1);
            if (lane == 31) eej = __ldg(a.rp + min(R1, rbj + TT));
            const int cntj = min(32, nsb - sb0);
            for (int j = 0; j < cntj; ++j) {
                const int eb = __shfl_sync(~0u, ebj, j), ee = __shfl_sync(~0u, eej, j);
                if (lane != 0) continue;
                const int q = (sb0 + j) % NT;
                const int rb = R0 + (sb0 + j) * TT, re = min(R1, rb + TT);
                const int a0 = eb & ~3;
                bool first = true;
                for (int cs = a0; cs < ee; cs += SE, first = false) {
                    while (rel[q] < iss[q] - S + 1) release_one(q);
                    const int slot = q * S + iss[q] % S;
                    const int len = min(SE, (ee - cs + 3) & ~3);
                    uint32_t tx = (uint32_t)len * 12;
                    int wnew = whi;
                    if (first) {
                        wnew = min(a.n, re + a.band);
                        if (M == 1) wnew = min(a.n, (wnew + 1) & ~1);
                        if (wnew > whi) {
                            // rows below wnew - WCAP are overwritten: every stage still in
                            // flight must belong to a sub-block starting at or above that + band
                            for (int t = 0; t < NT; ++t)
                                while (rel[t] < iss[t] && wnew - WCAP > slot_rb[t * S + rel[t] % S] - a.band)
                                    release_one(t);
                            tx += (uint32_t)(wnew - whi) * M * 8;
                        } else wnew = whi;
                    }
                    slot_rb[slot] = rb;
                    mb_expect(full + slot, tx);
                    unsigned char* st = ring + slot * STB;
                    bulk_g2s(st, a.ci + cs, (uint32_t)len * 4, full + slot);
                    bulk_g2s(st + SE * 4, a.v + cs, (uint32_t)len * 8, full + slot);
                    if (wnew > whi) {
                        int c = whi;
                        while (c < wnew) {             // split at the ring wrap and at 32 KB
                            const int sl = c % WCAP;
                            const int cnt = min(min(wnew - c, WCAP - sl), 32768 / (M * 8));
                            bulk_g2s(xs + (size_t)sl * M, a.x + (size_t)c * M, (uint32_t)cnt * M * 8, full + slot);
                            c += cnt;
                        }
                        whi = wnew;
                    }
                    iss[q] += 1;
                }
            }
        }
        return;
    }
    // ---------------- consumers
    const int team = threadIdx.x / TT, tt = threadIdx.x % TT;
    double* Pt = P + (size_t)team * PSZ * M;
    int it = 0;                                        // the team's stage counter
    for (int sb = team; sb < nsb; sb += NT) {
        const int rb = R0 + sb * TT, re = min(R1, rb + TT);
        const int eb = __ldg(a.rp + rb), ee = __ldg(a.rp + re);
        const int a0 = eb & ~3;
        const int row = rb + tt;
        int lo = 0, hi = 0;
        if (row < re) { lo = __ldg(a.rp + row); hi = __ldg(a.rp + row + 1); }
        const int wbase = max(0, rb - a.band) & ~1;    // lowest x row this sub-block may read
        const int wslot = wbase % WCAP;
        double acc[M];
#pragma unroll
        for (int i = 0; i < M; ++i) acc[i] = 0.0;
        for (int pb = a0; pb < ee; pb += PCAP) {       // product pieces (usually one per sub-block)
            const int pe = min(ee, pb + PCAP);
            for (int cs = pb; cs < pe; cs += SE, ++it) {
                const int slot = team * S + it % S;
                mb_wait(full + slot, (it / S) & 1);
                const uint32_t* sc = reinterpret_cast<const uint32_t*>(ring + slot * STB);
                const double* sv = reinterpret_cast<const double*>(ring + slot * STB + SE * 4);
                const int i0 = max(eb, cs) - cs, i1 = min(pe, cs + SE) - cs;
                constexpr int U1 = 4;
                for (int ib = i0 + tt; ib < i1; ib += TT * U1) {
                    int sl[U1]; double v[U1];
#pragma unroll
                    for (int u = 0; u < U1; ++u) {
                        const int i = min(ib + u * TT, i1 - 1);
                        sl[u] = wslot + ((int)sc[i] - wbase);
                        v[u] = sv[i];
                    }
                    fence();
                    double px[U1][M];
#pragma unroll
                    for (int u = 0; u < U1; ++u) {
                        if (sl[u] >= WCAP) sl[u] -= WCAP;
                        if constexpr (M == 1) px[u][0] = xs[sl[u]];
                        else {
                            const double2 t = *reinterpret_cast<const double2*>(xs + 2 * sl[u]);
                            px[u][0] = t.x; px[u][1] = t.y;
                        }
                    }
                    fence();
#pragma unroll
                    for (int u = 0; u < U1; ++u) {
                        const int i = ib + u * TT;
                        if (i < i1) {
                            const int q = ppos(cs - pb + i);
                            if constexpr (M == 1) Pt[q] = mul(v[u], px[u][0]);
                            else *reinterpret_cast<double2*>(Pt + 2 * q) =
                                     make_double2(mul(v[u], px[u][0]), mul(v[u], px[u][1]));
                        }
                    }
                }
                __syncwarp();
                if (threadIdx.x % 32 == 0) mb_arrive(empty + slot);
            }
            bar_team(1 + team, TT);
            const int klo = max(lo, pb) - pb, khi = min(hi, pe) - pb;
            constexpr int U2 = 4;
            for (int k = klo; k < khi; k += U2) {
                double t[U2][M];
#pragma unroll
                for (int u = 0; u < U2; ++u) {
                    const int kk = ppos(min(k + u, khi - 1));
                    if constexpr (M == 1) t[u][0] = Pt[kk];
                    else {
                        const double2 q = *reinterpret_cast<const double2*>(Pt + 2 * kk);
                        t[u][0] = q.x; t[u][1] = q.y;
                    }
                }
                fence();
#pragma unroll
                for (int u = 0; u < U2; ++u)
                    if (k + u < khi)
#pragma unroll
                        for (int i = 0; i < M; ++i) acc[i] = add(acc[i], t[u][i]);
            }
            bar_team(1 + team, TT);
        }
        if (row < re) {
            if constexpr (M == 1) a.y[row] = acc[0];
            else *reinterpret_cast<double2*>(a.y + 2 * (size_t)row) = make_double2(acc[0], acc[1]);
        }
    }
}


// ------------------------------------------------------------------ direct (m = 1, 2)
// The stream producer (entry ring per team + sliding x window) with thread-per-row
// consumers that accumulate straight from the staged entries (no product buffer):
// NT teams of TT threads; team q owns sub-blocks q, q + NT, ... and a private ring of ST
// slots that holds one whole sub-block.
template <int M, int TT, int NT, int LSE, int ST>
__global__ void __launch_bounds__(TT * NT + 32, 1) k_direct(S2Args a) {
    constexpr int T = TT * NT, SE = 1 << LSE, NS = ST * NT, STB = SE * 12;
    extern __shared__ __align__(128) unsigned char sm[];
    const int WCAP = a.wcap;
    double* xs = reinterpret_cast<double*>(sm);                              // WCAP x M
    unsigned char* ring = reinterpret_cast<unsigned char*>(xs + (size_t)WCAP * M);
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + NS * STB);
    uint64_t* empty = full + NS;
    int* slot_rb = reinterpret_cast<int*>(empty + NS);
    int* iss = slot_rb + NS;
    int* rel = iss + NT;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) { mb_init(full + s, 1); mb_init(empty + s, TT / 32); }
        for (int q = 0; q < NT; ++q) { iss[q] = 0; rel[q] = 0; }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int R0 = min(a.n, (int)blockIdx.x * a.rows_per_cta);
    const int R1 = min(a.n, R0 + a.rows_per_cta);
    if (R0 >= R1) return;
    const int nsb = (R1 - R0 + TT - 1) / TT;
    if (threadIdx.x >= T) {
        // ---------------- producer warp
        const int lane = threadIdx.x - T;
        int whi = max(0, R0 - a.band) & ~1;
        auto release_one = [&](int q) {
            const int r = rel[q];
            mb_wait(empty + q * ST + r % ST, (r / ST) & 1);
            rel[q] = r + 1;
        };
        for (int sb0 = 0; sb0 < nsb; sb0 += 32) {
            const int rbj = min(R1, R0 + (sb0 + lane) * TT);
            const int ebj = __ldg(a.rp + rbj);
            int eej = __shfl_down_sync(~0u, ebj, 1);
            if (lane == 31) eej = __ldg(a.rp + min(R1, rbj + TT));
            const int cntj = min(32, nsb - sb0);
            for (int j = 0; j < cntj; ++j) {
                const int eb = __shfl_sync(~0u, ebj, j), ee = __shfl_sync(~0u, eej, j);
                if (lane != 0) continue;
                const int q = (sb0 + j) % NT;
                const int rb = R0 + (sb0 + j) * TT, re = min(R1, rb + TT);
                bool first = true;
                for (int cs = eb & ~7; cs < ee; cs += SE, first = false) {
                    while (rel[q] < iss[q] - ST + 1) release_one(q);
                    const int slot = q * ST + iss[q] % ST;
                    const int len = min(SE, (ee - cs + 7) & ~7);
                    uint32_t tx = (uint32_t)len * 12;
                    int wnew = whi;
                    if (first) {
                        wnew = min(a.n, (re + a.band + 1) & ~1);
                        if (wnew > whi) {
                            for (int t = 0; t < NT; ++t)
                                while (rel[t] < iss[t] && wnew - WCAP > slot_rb[t * ST + rel[t] % ST] - a.band)
                                    release_one(t);
                            tx += (uint32_t)(wnew - whi) * M * 8;
                        } else wnew = whi;
                    }
                    slot_rb[slot] = rb;
                    mb_expect(full + slot, tx);
                    unsigned char* st = ring + slot * STB;
                    bulk_g2s(st, a.ci + cs, (uint32_t)len * 4, full + slot);
                    bulk_g2s(st + SE * 4, a.v + cs, (uint32_t)len * 8, full + slot);
                    for (int c = whi; c < wnew;) {
                        const int sl = c % WCAP;
                        const int cnt = min(min(wnew - c, WCAP - sl), 32768 / (M * 8));
                        bulk_g2s(xs + (size_t)sl * M, a.x + (size_t)c * M, (uint32_t)cnt * M * 8, full + slot);
                        c += cnt;
                    }
                    whi = wnew;
                    iss[q] += 1;
                }
            }
        }
        return;
    }
    // ---------------- consumers: one thread per row
    const int team = threadIdx.x / TT, tt = threadIdx.x % TT;
    int it = 0;
    for (int sb = team; sb < nsb; sb += NT) {
        const int rb = R0 + sb * TT, re = min(R1, rb + TT);
        const int row = rb + tt;
        const int eb = __ldg(a.rp + rb), ee = __ldg(a.rp + re);
        int lo = 0, hi = 0;
        if (row < re) { lo = __ldg(a.rp + row); hi = __ldg(a.rp + row + 1); }
        const int a0 = eb & ~7;
        const int nst = ee > a0 ? (ee - a0 + SE - 1) >> LSE : 0;
        const int wbase = max(0, rb - a.band) & ~1;
        const int wofs = wbase % WCAP - wbase;
        for (int j = 0; j < nst; ++j) mb_wait(full + team * ST + (it + j) % ST, ((it + j) / ST) & 1);
        double acc[M];
#pragma unroll
        for (int i = 0; i < M; ++i) acc[i] = 0.0;
        int e = lo;
        while (e < hi) {
            const int j = (e - a0) >> LSE;
            const int send = min(hi, a0 + ((j + 1) << LSE));           // entries of this stage
            const unsigned char* st = ring + (size_t)(team * ST + (it + j) % ST) * STB;
            const uint32_t* sc = reinterpret_cast<const uint32_t*>(st) - (a0 + (j << LSE));
            const double* sv = reinterpret_cast<const double*>(st + SE * 4) - (a0 + (j << LSE));
            constexpr int U = 4;
            for (; e < send; e += U) {
                int sl[U]; double v[U]; double px[U][M];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int k = min(e + u, send - 1);
                    sl[u] = wofs + (int)sc[k];
                    v[u] = sv[k];
                }
                fence();
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (sl[u] >= WCAP) sl[u] -= WCAP;
                    if constexpr (M == 1) px[u][0] = xs[sl[u]];
                    else {
                        const double2 t = *reinterpret_cast<const double2*>(xs + 2 * sl[u]);
                        px[u][0] = t.x; px[u][1] = t.y;
                    }
                }
                fence();
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (e + u < send)
#pragma unroll
                        for (int i = 0; i < M; ++i) acc[i] = add(acc[i], mul(v[u], px[u][i]));
            }
            e = send;
        }
        if (row < re) {
            if constexpr (M == 1) a.y[row] = acc[0];
            else *reinterpret_cast<double2*>(a.y + 2 * (size_t)row) = make_double2(acc[0], acc[1]);
        }
        bar_team(1 + team, TT);
        if (threadIdx.x % 32 == 0)
            for (int j = 0; j < nst; ++j) mb_arrive(empty + team * ST + (it + j) % ST);
        it += nst;
    }
}

// ------------------------------------------------------------------ tile (m >= 4)
// Band-tile format: rows in blocks of R, each block's column window cut into tiles
// of W columns; tile = packed [u16 ptr[R+8] | u16 col[ne] (tile-relative) | f64 val[ne]],
// entries of a tile in (row, column) order, so a row's entries are visited in CSR
// order as the tiles advance.  One persistent CTA per SM; per tile one TMA bulk copy
// of the packed matrix data and one of the W x-rows into a 2-stage shared-memory
// ring; a group of LPR lanes owns RG consecutive rows with accumulators in registers.
struct TileArgs {
    const int4* tiles;       // {off16, bytes, xcol0, xrows}
    const int2* blocks;      // {tile0, ntiles}
    const unsigned char* pack;
    const double* x;
    double* y;
    int n, nblocks, R, W, matb;   // matb: matrix bytes capacity per stage (16-aligned)
};


template <int M, int T, int RG>
__global__ void __launch_bounds__(T, 1) k_tile(TileArgs a) {
    constexpr int CPL = 2, LPR = M / CPL, S = 2;
    static_assert(RG == 8, "ptr vector load assumes 8 rows per group");
    extern __shared__ __align__(128) unsigned char sm[];
    const int stageb = a.matb + a.W * M * 8;
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + S * stageb);
    uint64_t* empty = full + S;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) { mb_init(full + s, 1); mb_init(empty + s, T / 32); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int g = threadIdx.x / LPR, lane = threadIdx.x % LPR;
    const int ptrb = (a.R + 8) * 2;
    // producer iterator (thread 0): next tile to issue
    int pI = blockIdx.x, pk = 0, pq = 0;
    int2 pblk = pI < a.nblocks ? a.blocks[pI] : make_int2(0, 0);
    auto issue = [&]() {        // thread 0 only
        if (pI >= a.nblocks) return;
        const int s = pq % S, use = pq / S;
        if (use > 0) mb_wait(empty + s, (use - 1) & 1);
        const int4 t = a.tiles[pblk.x + pk];
        unsigned char* st = sm + s * stageb;
        mb_expect(full + s, (uint32_t)t.y + (uint32_t)t.w * M * 8);
        bulk_g2s(st, a.pack + (size_t)t.x * 16, (uint32_t)t.y, full + s);
        const uint32_t xb = (uint32_t)t.w * M * 8;
        const unsigned char* xsrc = reinterpret_cast<const unsigned char*>(a.x + (size_t)t.z * M);
        for (uint32_t off = 0; off < xb; off += 32768)
            bulk_g2s(st + a.matb + off, xsrc + off, min(xb - off, 32768u), full + s);
        ++pq;
        if (++pk == pblk.y) {
            pk = 0;
            pI += gridDim.x;
            if (pI < a.nblocks) pblk = a.blocks[pI];
        }
    };
    if (threadIdx.x == 0) issue();
    int q = 0;
    for (int I = blockIdx.x; I < a.nblocks; I += gridDim.x) {
        const int2 blk = a.blocks[I];
        double acc[RG][CPL];
#pragma unroll
        for (int j = 0; j < RG; ++j) { acc[j][0] = 0.0; acc[j][1] = 0.0; }
        for (int k = 0; k < blk.y; ++k, ++q) {
            if (threadIdx.x == 0) issue();          // tile q+1 into the other stage
            __syncwarp();
            const int s = q % S;
            mb_wait(full + s, (q / S) & 1);
            const unsigned char* st = sm + s * stageb;
            const uint16_t* ptr = reinterpret_cast<const uint16_t*>(st);
            const int ne = ptr[a.R];
            const uint16_t* cols = reinterpret_cast<const uint16_t*>(st + ptrb);
            const double* vals = reinterpret_cast<const double*>(st + ptrb + ((ne * 2 + 15) & ~15));
            const double* xs = reinterpret_cast<const double*>(st + a.matb) + lane * CPL;
            const uint4 pw = *reinterpret_cast<const uint4*>(ptr + g * RG);
            int p[RG + 1];
            p[0] = pw.x & 0xffff; p[1] = pw.x >> 16; p[2] = pw.y & 0xffff; p[3] = pw.y >> 16;
            p[4] = pw.z & 0xffff; p[5] = pw.z >> 16; p[6] = pw.w & 0xffff; p[7] = pw.w >> 16;
            p[8] = ptr[g * RG + 8];
#pragma unroll
            for (int j = 0; j < RG; ++j) {
                for (int e = p[j]; e < p[j + 1]; ++e) {
                    const int c = cols[e];
                    const double v = vals[e];
                    const double2 xv = *reinterpret_cast<const double2*>(xs + c * M);
                    acc[j][0] = add(acc[j][0], mul(v, xv.x));
                    acc[j][1] = add(acc[j][1], mul(v, xv.y));
                }
            }
            __syncwarp();
            if (threadIdx.x % 32 == 0) mb_arrive(empty + s);
        }
        const int r0 = I * a.R + g * RG;
#pragma unroll
        for (int j = 0; j < RG; ++j)
            if (r0 + j < a.n)
                *reinterpret_cast<double2*>(a.y + (size_t)(r0 + j) * M + lane * CPL) =
                    make_double2(acc[j][0], acc[j][1]);
    }
}

// ------------------------------------------------------------------ host
struct Csr {
    int n;
    std::vector<int> rp;
    std::vector<uint32_t> ci;
    std::vector<double> v;
};

static Csr band_random(int n, int band, double mean) {
    Csr A;
    A.n = n;
    std::mt19937_64 rng(5);
    std::poisson_distribution<int> P(mean / 2);
    std::uniform_int_distribution<int> D(1, band);
    std::normal_distribution<double> N(0, 1);
    std::vector<std::vector<std::pair<int, double>>> rows(n);
    for (int i = 0; i < n; ++i) {
        int k = P(rng);
        for (int t = 0; t < k; ++t) {
            int j = i + D(rng);
            if (j >= n) continue;
            double w = N(rng);
            rows[i].push_back({j, w});
            rows[j].push_back({i, w});
        }
    }
    A.rp.push_back(0);
    for (int i = 0; i < n; ++i) {
        auto& r = rows[i];
        r.push_back({i, 0.0});
        std::sort(r.begin(), r.end());
        int w = 0;
        for (size_t t = 0; t < r.size(); ++t) {
            if (w && r[w - 1].first == r[t].first) { r[w - 1].second += r[t].second; continue; }
            r[w++] = r[t];
        }
        r.resize(w);
        double s = 1;
        for (auto& e : r) s += fabs(e.second);
        for (auto& e : r) {
            A.ci.push_back(e.first);
            A.v.push_back(e.first == i ? s : e.second);
        }
        A.rp.push_back((int)A.ci.size());
        std::vector<std::pair<int, double>>().swap(r);
    }
    return A;
}


struct TileFmt {
    std::vector<int4> tiles;
    std::vector<int2> blocks;
    std::vector<unsigned char> pack;
    int R, W, matb, max_ne;
};

static TileFmt build_tiles(const Csr& A, int R, int W) {
    TileFmt F;
    F.R = R; F.W = W; F.max_ne = 0;
    const int nb = (A.n + R - 1) / R;
    const int ptrb = (R + 8) * 2;
    std::vector<int> cnt;
    for (int I = 0; I < nb; ++I) {
        const int r0 = I * R, r1 = std::min(A.n, r0 + R);
        uint32_t mn = UINT32_MAX, mx = 0;
        for (int k = A.rp[r0]; k < A.rp[r1]; ++k) { mn = std::min(mn, A.ci[k]); mx = std::max(mx, A.ci[k]); }
        if (mn == UINT32_MAX) { mn = 0; mx = 0; }
        const int cb = (int)(mn & ~15u);
        const int nt = (int)((mx - cb) / W) + 1;
        F.blocks.push_back(make_int2((int)F.tiles.size(), nt));
        // per (tile, row) counts
        cnt.assign((size_t)nt * (R + 1), 0);
        for (int r = r0; r < r1; ++r)
            for (int k = A.rp[r]; k < A.rp[r + 1]; ++k) cnt[(size_t)((A.ci[k] - cb) / W) * (R + 1) + (r - r0) + 1]++;
        for (int t = 0; t < nt; ++t) {
            int* c = cnt.data() + (size_t)t * (R + 1);
            for (int j = 0; j < R; ++j) c[j + 1] += c[j];
            const int ne = c[R];
            F.max_ne = std::max(F.max_ne, ne);
            const size_t colb = ((size_t)ne * 2 + 15) & ~(size_t)15, valb = ((size_t)ne * 8 + 15) & ~(size_t)15;
            const size_t off = F.pack.size();
            F.pack.resize(off + ptrb + colb + valb, 0);
            uint16_t* ptr = reinterpret_cast<uint16_t*>(F.pack.data() + off);
            for (int j = 0; j <= R; ++j) ptr[j] = (uint16_t)c[j];
            for (int j = R + 1; j < R + 8; ++j) ptr[j] = (uint16_t)ne;
            const int xcol0 = cb + t * W;
            F.tiles.push_back(make_int4((int)(off / 16), (int)(ptrb + colb + valb), xcol0, std::min(W, A.n - xcol0)));
        }
        // fill entries: rows in order, each row's entries in column order
        std::vector<int> pos(nt, 0);
        for (int r = r0; r < r1; ++r)
            for (int k = A.rp[r]; k < A.rp[r + 1]; ++k) {
                const int t = (int)((A.ci[k] - cb) / W);
                const int4 ti = F.tiles[F.blocks.back().x + t];
                unsigned char* base = F.pack.data() + (size_t)ti.x * 16;
                const int ne = reinterpret_cast<uint16_t*>(base)[R];
                uint16_t* cols = reinterpret_cast<uint16_t*>(base + ptrb);
                double* vals = reinterpret_cast<double*>(base + ptrb + (((size_t)ne * 2 + 15) & ~(size_t)15));
                cols[pos[t]] = (uint16_t)(A.ci[k] - ti.z);
                vals[pos[t]] = A.v[k];
                pos[t]++;
            }
    }
    F.matb = (int)((ptrb + (((size_t)F.max_ne * 2 + 15) & ~(size_t)15) + (size_t)F.max_ne * 8 + 15) & ~(size_t)15);
    return F;
}

template <typename T> static T* up(const std::vector<T>& h, size_t pad = 64) {
    T* d;
    CK(cudaMalloc(&d, (h.size() + pad) * sizeof(T)));
    CK(cudaMemset(d, 0, (h.size() + pad) * sizeof(T)));
    CK(cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
    return d;
}

static double* g_flush;
static void flush_l2() { CK(cudaMemsetAsync(g_flush, 0, 256u << 20)); }

template <class F> static float time_us(F&& f, int reps = 11) {
    std::vector<float> ts;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int r = 0; r < reps; ++r) {
        flush_l2();
        cudaEventRecord(e0);
        f();
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        ts.push_back(ms * 1e3f);
    }
    CK(cudaGetLastError());
    std::sort(ts.begin(), ts.end());
    return ts[ts.size() / 2];
}

static int nsm() { int v; cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, 0); return v; }

static std::vector<double> g_ref;
static bool want(const char* name) {
    const char* sel = getenv("BP_SEL");
    return !sel || strstr(name, sel) || !strncmp(name, "lane", 4);
}
static void check(const char* name, const double* dy, size_t cnt, float us, double bytes) {
    std::vector<double> h(cnt);
    CK(cudaMemcpy(h.data(), dy, cnt * 8, cudaMemcpyDeviceToHost));
    const char* st = "first";
    if (g_ref.empty()) g_ref = h;
    else st = memcmp(g_ref.data(), h.data(), cnt * 8) == 0 ? "bitwise" : "MISMATCH";
    printf("  %-28s %9.1f us  %7.1f GB/s  %s\n", name, us, bytes / us * 1e-3, st);
    fflush(stdout);
    CK(cudaMemset((void*)dy, 0xff, cnt * 8));
}

template <int M> static void bench(const Csr& A, int band) {
    constexpr int LPR = Lay<M>::LPR, RPB = 256 / LPR;
    const size_t nnz = A.ci.size();
    Args a = {};
    a.rp = up(A.rp); a.ci = up(A.ci); a.v = up(A.v);
    a.n = A.n; a.band = band;
    std::vector<double> hx((size_t)A.n * M);
    std::mt19937_64 rng(7);
    std::uniform_real_distribution<double> U(-1, 1);
    for (auto& t : hx) t = U(rng);
    a.x = up(hx);
    double* y;
    CK(cudaMalloc(&y, (size_t)A.n * M * 8));
    a.y = y;
    const double bytes = nnz * 12.0 + (A.n + 1) * 4.0 + 2.0 * A.n * M * 8;
    printf("m = %d   n = %d  nnz = %zu  algorithmic %.1f MB\n", M, A.n, nnz, bytes * 1e-6);
    g_ref.clear();
    const int S = nsm();
    {   // lane (library design)
        auto kern = k_lane<M, 4, 6>;
        int bps;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, 256, 0);
        const long cap = (long)bps * S;
        const long P = (a.n + RPB - 1) / RPB, ppc = (P + cap - 1) / cap;
        const long pmax = RPB >= 64 ? 1 : 64 / RPB;
        const long sp = std::min(ppc, pmax);
        const long nch = (P + sp - 1) / sp, cpc = (nch + cap - 1) / cap;
        const int grid = (int)((nch + cpc - 1) / cpc);
        a.chunk = (int)(RPB * sp);
        float us = time_us([&] { kern<<<grid, 256>>>(a); });
        check("lane (64-row chunks, strided)", y, (size_t)A.n * M, us, bytes);
    }
    auto remap = [&](auto kern, const char* name, int chunk) {
        if (!want(name)) return;
        int bps;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, 256, 0);
        a.nsm = S; a.cps = bps; a.chunk = chunk;
        float us = time_us([&] { kern<<<S * bps, 256>>>(a); });
        char buf[96];
        snprintf(buf, sizeof buf, "%s chunk %d x%d", name, chunk, bps);
        check(buf, y, (size_t)A.n * M, us, bytes);
    };
    for (int ch : {RPB, 4 * RPB}) {
        remap(k_remap<M, 4, 6, 0>, "remap", ch);
        remap(k_remap<M, 4, 6, 1>, "remap na", ch);
    }
    remap(k_remap<M, 4, 4, 1>, "remap na occ4", RPB);
    remap(k_remap<M, 4, 3, 1>, "remap na occ3", RPB);
    if constexpr (M <= 2) {
        auto stream = [&](auto kern, int T, int PE, int R, const char* name) {
            if (!want(name)) return;
            a.R = R;
            a.nblocks = (A.n + R - 1) / R;
            const size_t smem = ((size_t)(R + 2 * band + 2) * M + (size_t)PE * M) * 8 + 16;
            if (smem > 227 * 1024) { printf("  %s: smem %zu too large\n", name, smem); return; }
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            int bps;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, T, smem);
            const int grid = std::min(a.nblocks, bps * S);
            float us = time_us([&] { kern<<<grid, T, smem>>>(a); });
            char buf[96];
            snprintf(buf, sizeof buf, "%s R %d x%d (%zu KB)", name, R, bps, smem >> 10);
            check(buf, y, (size_t)A.n * M, us, bytes);
        };


        auto direct = [&](auto kern, int TT, int NT, int LSE, int ST, const char* name) {
            if (!want(name)) return;
            const int SE = 1 << LSE;
            S2Args t = {};
            t.rp = a.rp; t.ci = a.ci; t.v = a.v; t.x = a.x; t.y = y; t.n = A.n; t.band = band;
            t.wcap = (2 * band + (NT + 1) * TT + 256 + 1) & ~1;
            const int grid = S;
            t.rows_per_cta = (((A.n + grid - 1) / grid + TT - 1) / TT) * TT;
            int mxs = 0;
            for (int r = 0; r < A.n; r += TT) {
                const int eb = A.rp[r], ee = A.rp[std::min(A.n, r + TT)];
                if (ee > (eb & ~7)) mxs = std::max(mxs, (ee - (eb & ~7) + SE - 1) / SE);
            }
            if (mxs > ST) { printf("  %s: a sub-block needs %d stages > %d\n", name, mxs, ST); return; }
            const size_t smem = (size_t)t.wcap * M * 8 + (size_t)ST * NT * SE * 12 + ST * NT * 20 + NT * 8 + 16;
            if (smem > 227 * 1024) { printf("  %s: smem %zu too large\n", name, smem); return; }
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            float us = time_us([&] { kern<<<grid, TT * NT + 32, smem>>>(t); });
            char buf[128];
            snprintf(buf, sizeof buf, "%s TT%d NT%d SE%d ST%d (%zuK)", name, TT, NT, SE, ST, smem >> 10);
            check(buf, y, (size_t)A.n * M, us, bytes);
        };
        if constexpr (M == 1) {
            direct(k_direct<M, 256, 2, 10, 6>, 256, 2, 10, 6, "direct-a");
            direct(k_direct<M, 128, 4, 9, 6>, 128, 4, 9, 6, "direct-b");
            direct(k_direct<M, 128, 3, 9, 6>, 128, 3, 9, 6, "direct-c");
            direct(k_direct<M, 256, 1, 10, 8>, 256, 1, 10, 8, "direct-d");
            direct(k_direct<M, 192, 3, 9, 8>, 192, 3, 9, 8, "direct-e");
        } else {
            direct(k_direct<M, 128, 2, 9, 6>, 128, 2, 9, 6, "direct-a");
            direct(k_direct<M, 64, 4, 8, 6>, 64, 4, 8, 6, "direct-b");
            direct(k_direct<M, 96, 3, 8, 8>, 96, 3, 8, 8, "direct-c");
            direct(k_direct<M, 128, 1, 9, 12>, 128, 1, 9, 12, "direct-d");
        }
        auto stream3 = [&](auto kern, int TT, int NT, int SE, int Sg, int PCAP, int wcap, const char* name) {
            if (!want(name)) return;
            S2Args t = {};
            t.rp = a.rp; t.ci = a.ci; t.v = a.v; t.x = a.x; t.y = y; t.n = A.n; t.band = band; t.wcap = wcap;
            const int grid = S;
            t.rows_per_cta = (((A.n + grid - 1) / grid + TT - 1) / TT) * TT;
            const size_t smem = ((size_t)wcap * M + (size_t)(PCAP + PCAP / 16 + 2) * M * NT) * 8 + (size_t)Sg * NT * SE * 12 + Sg * NT * 20 + NT * 8 + 16;
            if (smem > 227 * 1024) { printf("  %s: smem %zu too large\n", name, smem); return; }
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            float us = time_us([&] { kern<<<grid, TT * NT + 32, smem>>>(t); });
            char buf[128];
            snprintf(buf, sizeof buf, "%s TT%d NT%d SE%d S%d P%d (%zuK)", name, TT, NT, SE, Sg, PCAP, smem >> 10);
            check(buf, y, (size_t)A.n * M, us, bytes);
        };
        auto stream6 = [&](auto kern, int T, int NP, int SE, int Sg, int PCAP, int wcap, const char* name) {
            if (!want(name)) return;
            S2Args t = {};
            t.rp = a.rp; t.ci = a.ci; t.v = a.v; t.x = a.x; t.y = y; t.n = A.n; t.band = band; t.wcap = wcap;
            const int grid = S;
            t.rows_per_cta = (((A.n + grid - 1) / grid + T - 1) / T) * T;
            int mx = 0;
            for (int r = 0; r < A.n; r += T) mx = std::max(mx, A.rp[std::min(A.n, r + T)] - A.rp[r]);
            if (mx + 3 > PCAP) { printf("  %s: sub-block of %d entries > PCAP\n", name, mx); return; }
            const size_t smem = ((size_t)wcap * M + (size_t)PCAP * M * 2) * 8 + (size_t)Sg * SE * 12 + Sg * 16 + 32 + Sg * 4 + 16;
            if (smem > 227 * 1024) { printf("  %s: smem %zu too large\n", name, smem); return; }
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            float us = time_us([&] { kern<<<grid, T + NP + 32, smem>>>(t); });
            char buf[128];
            snprintf(buf, sizeof buf, "%s T%d NP%d SE%d S%d P%d (%zuK)", name, T, NP, SE, Sg, PCAP, smem >> 10);
            check(buf, y, (size_t)A.n * M, us, bytes);
        };
        auto stream5 = [&](auto kern, int T, int SE, int Sg, int PCAP, int wcap, const char* name) {
            if (!want(name)) return;
            S2Args t = {};
            t.rp = a.rp; t.ci = a.ci; t.v = a.v; t.x = a.x; t.y = y; t.n = A.n; t.band = band; t.wcap = wcap;
            const int grid = S;
            t.rows_per_cta = (((A.n + grid - 1) / grid + T - 1) / T) * T;
            int mx = 0;
            for (int r = 0; r < A.n; r += T) mx = std::max(mx, A.rp[std::min(A.n, r + T)] - A.rp[r]);
            if (mx + 3 > PCAP) { printf("  %s: sub-block of %d entries > PCAP\n", name, mx); return; }
            const size_t smem = ((size_t)wcap * M + (size_t)PCAP * M * 2) * 8 + (size_t)Sg * SE * 12 + Sg * 16 + Sg * 4 + 16;
            if (smem > 227 * 1024) { printf("  %s: smem %zu too large\n", name, smem); return; }
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            float us = time_us([&] { kern<<<grid, T + 32, smem>>>(t); });
            char buf[128];
            snprintf(buf, sizeof buf, "%s T%d SE%d S%d P%d (max sb %d; %zuK)", name, T, SE, Sg, PCAP, mx, smem >> 10);
            check(buf, y, (size_t)A.n * M, us, bytes);
        };
        auto stream2 = [&](auto kern, int T, int SE, int Sg, int PCAP, int wcap, const char* name, int pf = 0) {
            if (!want(name)) return;
            S2Args t = {};
            t.rp = a.rp; t.ci = a.ci; t.v = a.v; t.x = a.x; t.y = y; t.n = A.n; t.band = band; t.wcap = wcap; t.pf_entries = pf;
            const int grid = S;
            t.rows_per_cta = (((A.n + grid - 1) / grid + T - 1) / T) * T;
            const size_t smem = ((size_t)wcap * M + (size_t)PCAP * M) * 8 + (size_t)Sg * SE * 12 + Sg * 16 + Sg * 4 + 16;
            if (smem > 227 * 1024) { printf("  %s: smem %zu too large\n", name, smem); return; }
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            float us = time_us([&] { kern<<<grid, T + 32, smem>>>(t); });
            char buf[128];
            snprintf(buf, sizeof buf, "%s T%d SE%d S%d P%d W%d pf%d (%zuK)", name, T, SE, Sg, PCAP, wcap, pf, smem >> 10);
            check(buf, y, (size_t)A.n * M, us, bytes);
        };
        if constexpr (M == 1) {
            stream2(k_stream2<M, 256, 2048, 4, 6144>, 256, 2048, 4, 6144, 9728, "stream2a");
            stream2(k_stream2<M, 512, 2048, 2, 10240>, 512, 2048, 2, 10240, 9728, "stream2b");
            stream2(k_stream2<M, 512, 1024, 4, 10240>, 512, 1024, 4, 10240, 9728, "stream2c");
            stream2(k_stream2<M, 384, 1024, 6, 8192>, 384, 1024, 6, 8192, 9728, "stream2d");
            stream2(k_stream2<M, 640, 512, 4, 12288>, 640, 512, 4, 12288, 9728, "stream2e");
            stream3(k_stream3<M, 256, 1, 1024, 8, 5120>, 256, 1, 1024, 8, 5120, 9728, "stream3a");
            stream3(k_stream3<M, 256, 2, 512, 5, 5120>, 256, 2, 512, 5, 5120, 9728, "stream3b");
            stream3(k_stream3<M, 256, 2, 1024, 3, 4096>, 256, 2, 1024, 3, 4096, 9728, "stream3c");
            stream3(k_stream3<M, 128, 4, 512, 3, 2560>, 128, 4, 512, 3, 2560, 9728, "stream3d");
            stream3(k_stream3<M, 128, 3, 512, 4, 2560>, 128, 3, 512, 4, 2560, 9728, "stream3e");
            stream3(k_stream3<M, 192, 3, 512, 3, 3584>, 192, 3, 512, 3, 3584, 9728, "stream3f");
            stream3(k_stream3<M, 128, 6, 256, 4, 2560>, 128, 6, 256, 4, 2560, 9728, "stream3g");
            stream6(k_stream6<M, 256, 128, 2048, 3, 4608>, 256, 128, 2048, 3, 4608, 8704, "stream8a");
            stream6(k_stream6<M, 256, 128, 1536, 4, 4608>, 256, 128, 1536, 4, 4608, 8704, "stream8b");
            stream6(k_stream6<M, 256, 192, 2048, 3, 4608>, 256, 192, 2048, 3, 4608, 8704, "stream8c");
            stream6(k_stream6<M, 256, 192, 3072, 2, 4608>, 256, 192, 3072, 2, 4608, 8704, "stream8d");
            stream6(k_stream6<M, 256, 96, 1536, 4, 4608>, 256, 96, 1536, 4, 4608, 8704, "stream8e");
            stream6(k_stream6<M, 256, 160, 1280, 5, 4608>, 256, 160, 1280, 5, 4608, 8704, "stream8f");
            stream6(k_stream6<M, 256, 192, 1152, 5, 4608>, 256, 192, 1152, 5, 4608, 8704, "stream8g");
            stream6(k_stream6<M, 256, 384, 1536, 4, 4608>, 256, 384, 1536, 4, 4608, 8704, "stream7a");
            stream6(k_stream6<M, 256, 384, 768, 8, 4608>, 256, 384, 768, 8, 4608, 8704, "stream7b");
            stream6(k_stream6<M, 256, 320, 1280, 5, 4608>, 256, 320, 1280, 5, 4608, 8704, "stream7c");
            stream6(k_stream6<M, 256, 448, 1792, 3, 4608>, 256, 448, 1792, 3, 4608, 8704, "stream7d");
            stream6(k_stream6<M, 256, 256, 2048, 3, 4608>, 256, 256, 2048, 3, 4608, 8704, "stream7e");
            stream6(k_stream6<M, 256, 192, 1536, 4, 4608>, 256, 192, 1536, 4, 4608, 8704, "stream7f");
            stream6(k_stream6<M, 320, 384, 1536, 3, 5632>, 320, 384, 1536, 3, 5632, 8704, "stream7g");
            stream6(k_stream6<M, 256, 256, 1024, 5, 5120>, 256, 256, 1024, 5, 5120, 9728, "stream6a");
            stream6(k_stream6<M, 256, 512, 1024, 5, 5120>, 256, 512, 1024, 5, 5120, 9728, "stream6b");
            stream6(k_stream6<M, 256, 512, 2048, 2, 5120>, 256, 512, 2048, 2, 5120, 9728, "stream6c");
            stream6(k_stream6<M, 256, 384, 1536, 3, 5120>, 256, 384, 1536, 3, 5120, 9728, "stream6d");
            stream6(k_stream6<M, 192, 512, 1024, 7, 3840>, 192, 512, 1024, 7, 3840, 9728, "stream6e");
            stream6(k_stream6<M, 128, 512, 1024, 9, 2560>, 128, 512, 1024, 9, 2560, 9728, "stream6f");
            stream5(k_stream5<M, 256, 1024, 5, 5120>, 256, 1024, 5, 5120, 9728, "stream5a");
            stream5(k_stream5<M, 256, 512, 11, 4864>, 256, 512, 11, 4864, 9728, "stream5b");
            stream5(k_stream5<M, 192, 1024, 7, 3840>, 192, 1024, 7, 3840, 9728, "stream5c");
            stream5(k_stream5<M, 224, 1024, 6, 4352>, 224, 1024, 6, 4352, 9728, "stream5d");
            stream5(k_stream5<M, 160, 1024, 9, 3072>, 160, 1024, 9, 3072, 9728, "stream5e");
            stream2(k_stream4<M, 256, 2048, 4, 6144>, 256, 2048, 4, 6144, 9728, "stream4a");
            stream2(k_stream4<M, 256, 2048, 4, 6144>, 256, 2048, 4, 6144, 9728, "stream4a-nocompute", -1);
            stream2(k_stream4<M, 256, 2048, 4, 6144>, 256, 2048, 4, 6144, 9728, "stream4a-nophase2", -2);
            stream2(k_stream4<M, 256, 1024, 8, 6144>, 256, 1024, 8, 6144, 9728, "stream4b");
            stream2(k_stream4<M, 384, 1024, 6, 8192>, 384, 1024, 6, 8192, 9728, "stream4d");
            stream2(k_stream4<M, 320, 1024, 7, 7168>, 320, 1024, 7, 7168, 9728, "stream4e");
            for (int pf : {8192}) {
                stream2(k_stream2<M, 256, 2048, 4, 6144>, 256, 2048, 4, 6144, 9728, "stream2f", pf);
                stream2(k_stream2<M, 512, 1024, 4, 10240>, 512, 1024, 4, 10240, 9728, "stream2g", pf);
                stream2(k_stream2<M, 640, 512, 4, 12288>, 640, 512, 4, 12288, 9728, "stream2h", pf);
            }
        } else {
            stream2(k_stream2<M, 128, 1024, 3, 3072>, 128, 1024, 3, 3072, 9216, "stream2");
            stream2(k_stream2<M, 128, 512, 6, 3072>, 128, 512, 6, 3072, 9216, "stream2");
            stream2(k_stream2<M, 64, 512, 8, 1536>, 64, 512, 8, 1536, 9216, "stream2");
        }
        if constexpr (M == 1) {
            stream(k_stream<M, 512, 10240, 4>, 512, 10240, 2048, "stream T512 PE10k");
            stream(k_stream<M, 512, 10240, 4>, 512, 10240, 4096, "stream T512 PE10k");
            stream(k_stream<M, 1024, 20480, 4>, 1024, 20480, 8192, "stream T1024 PE20k");
            stream(k_stream<M, 256, 5120, 4>, 256, 5120, 1024, "stream T256 PE5k");
            stream(k_stream<M, 256, 5120, 8>, 256, 5120, 2048, "stream T256 PE5k u8");
        } else {
            stream(k_stream<M, 512, 5120, 4>, 512, 5120, 1024, "stream T512 PE5k");
            stream(k_stream<M, 512, 5120, 4>, 512, 5120, 2048, "stream T512 PE5k");
            stream(k_stream<M, 256, 5120, 4>, 256, 5120, 512, "stream T256 PE5k");
            stream(k_stream<M, 1024, 3072, 2>, 1024, 3072, 3072, "stream T1024 PE3k");
        }
    }

    if constexpr (M >= 4) {
        auto tile = [&](auto kern, int T, int R, int W, const char* name) {
            if (!want(name)) return;
            TileFmt F = build_tiles(A, R, W);
            const size_t smem = 2 * ((size_t)F.matb + (size_t)W * M * 8) + 64;
            printf("  [tile fmt R %d W %d: %zu tiles, %.1f MB packed, max_ne %d, smem %zu]\n", R, W,
                   F.tiles.size(), F.pack.size() * 1e-6, F.max_ne, smem);
            if (smem > 227 * 1024) { printf("  %s: smem too large\n", name); return; }
            TileArgs t = {};
            t.tiles = up(F.tiles); t.blocks = up(F.blocks); t.pack = up(F.pack);
            t.x = a.x; t.y = y; t.n = A.n; t.nblocks = (int)F.blocks.size(); t.R = R; t.W = W; t.matb = F.matb;
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            const int grid = std::min(t.nblocks, S);
            float us = time_us([&] { kern<<<grid, T, smem>>>(t); });
            char buf[96];
            snprintf(buf, sizeof buf, "%s R %d W %d", name, R, W);
            check(buf, y, (size_t)A.n * M, us, bytes);
            cudaFree((void*)t.tiles); cudaFree((void*)t.blocks); cudaFree((void*)t.pack);
        };
        constexpr int G = 1024 / (M / 2);
        if constexpr (M == 8) {
            tile(k_tile<M, 1024, 8>, 1024, G * 8, 896, "tile T1024");
            tile(k_tile<M, 1024, 8>, 1024, G * 8, 768, "tile T1024");
        } else if constexpr (M == 4) {
            tile(k_tile<M, 1024, 8>, 1024, G * 8, 1536, "tile T1024");
            tile(k_tile<M, 512, 8>, 512, G * 4, 2048, "tile T512");
        } else if constexpr (M == 16) {
            tile(k_tile<M, 1024, 8>, 1024, G * 8, 512, "tile T1024");
        }
    }
    cudaFree((void*)a.rp); cudaFree((void*)a.ci); cudaFree((void*)a.v); cudaFree((void*)a.x); cudaFree(y);
}

int main(int argc, char** argv) {
    CK(cudaMalloc(&g_flush, 256u << 20));
    const int lg = argc > 2 ? atoi(argv[2]) : 22;
    const int band = 4096;
    Csr A = band_random(1 << lg, band, 15.0);
    const int m = argc > 1 ? atoi(argv[1]) : 0;
    if (m == 0 || m == 1) bench<1>(A, band);
    if (m == 0 || m == 2) bench<2>(A, band);
    if (m == 0 || m == 4) bench<4>(A, band);
    if (m == 0 || m == 8) bench<8>(A, band);
    if (m == 0 || m == 16) bench<16>(A, band);
    return 0;
}
