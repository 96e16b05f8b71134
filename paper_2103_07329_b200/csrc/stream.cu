// stream.cu -- single-RHS (m = 1) SpMV for banded operators: the "stream" variant
// of csr_spmv (_ckernels.pyx:30-57), SpmmVariant SV_STREAM.
//
// Why: with one right-hand side the lane kernel (spmm.cuh) is one thread per row --
// every CSR load of a warp touches 32 different lines and every gathered x value
// costs a 32-byte sector from L2 (C5, n = 2^22, ~16 entries/row, columns within
// +-4096 of the diagonal: 377 us = 0.36 of the measured HBM peak).  When the
// operator's band fits shared memory the whole product can be fed by TMA instead:
//
//   * one persistent CTA per SM owns a contiguous row range;
//   * a producer warp streams the range's CSR entries (columns, values) through a
//     ring of shared-memory stages with cp.async.bulk (mbarrier complete_tx) and
//     keeps a sliding window of x rows -- a ring of WCAP values covering
//     [row - band, row + band] of every row in flight -- ahead of the consumers;
//   * product warps turn each stage into products P[e] = v_e * x[col_e], entry
//     parallel: perfectly coalesced matrix stream, gathers from shared memory;
//   * sum warps (one thread per row of a 256-row sub-block) add the row's products
//     in CSR entry order -- separately rounded multiply, then add/sub: bitwise the
//     reference kernel and the lane path;
//   * two product buffers are handed between product and sum warps with mbarriers,
//     so the ordered sums of sub-block s overlap the products of sub-block s + 1.
//
// C5 at m = 1: 208 us (0.65 of the measured peak), profiles/r02_band_probe.txt.
// Design notes and the rejected alternatives: scripts/probe/band_probe.cu.
#include <algorithm>
#include <atomic>
#include <cstdint>

#include "dispatch.h"

namespace mrs {

namespace {

constexpr int kSumT = 256;        // sum threads = rows per sub-block
constexpr int kProdT = 192;       // product threads
constexpr int kSE = 1536;         // entries per ring stage
constexpr int kPcap = 4608;       // product buffer capacity (entries of one sub-block + alignment)
constexpr int kAlign = 8;         // stages start at entry indices aligned to 8 (16 bytes of u16)

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

struct StArgs {
    const int32_t* rp;
    const void* ci;
    const void* vals;
    const int32_t* slab_base;   // non-null: column = slab_base[row >> slab_shift] + c16
    int slab_shift;
    const double* x;
    const double* b;
    double* y;
    int n, ncols, band, rows_per_cta, wcap, mode;
};

// Shared memory: x window (wcap doubles) | P[2][kPcap] | ring S x (cols | vals) |
// full[S], empty[S], pfull[2], pempty[2] | slot_rb[S] (producer-private).
template <typename Tv, typename Ti, int S>
__global__ void __launch_bounds__(kSumT + kProdT + 32, 1) stream_spmv_kernel(StArgs a) {
    constexpr int T = kSumT, NP = kProdT, SE = kSE, PCAP = kPcap;
    constexpr int STB = SE * (int)(sizeof(Ti) + sizeof(Tv));
    extern __shared__ __align__(128) unsigned char sm[];
    const int WCAP = a.wcap;
    double* xs = reinterpret_cast<double*>(sm);
    double* P = xs + WCAP;
    unsigned char* ring = reinterpret_cast<unsigned char*>(P + 2 * PCAP);
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + S * STB);
    uint64_t* empty = full + S;
    uint64_t* pfull = empty + S;
    uint64_t* pempty = pfull + 2;
    int* slot_rb = reinterpret_cast<int*>(pempty + 2);
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
    const Ti* gci = reinterpret_cast<const Ti*>(a.ci);
    const Tv* gv = reinterpret_cast<const Tv*>(a.vals);

    if (threadIdx.x >= T + NP) {
        // ---------------- producer warp (lane 0 issues; all lanes fetch row pointers)
        const int lane = threadIdx.x - T - NP;
        int issued = 0, released = 0;
        int whi = max(0, R0 - a.band) & ~1;            // x rows below whi are loaded (or on their way)
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
                bool first = true;
                for (int cs = eb & ~(kAlign - 1); cs < ee; cs += SE, first = false) {
                    const int slot = issued % S;
                    while (released < issued - S + 1) {
                        mb_wait(empty + released % S, (released / S) & 1);
                        ++released;
                    }
                    const int len = min(SE, (ee - cs + kAlign - 1) & ~(kAlign - 1));
                    uint32_t tx = (uint32_t)len * (uint32_t)(sizeof(Ti) + sizeof(Tv));
                    int wnew = whi;
                    if (first) {
                        wnew = min(a.ncols, (re + a.band + 1) & ~1);
                        if (wnew > whi) {
                            // the new rows overwrite rows below wnew - WCAP: every stage still
                            // in flight must belong to a sub-block that no longer reads them
                            while (released < issued && wnew - WCAP > slot_rb[released % S] - a.band) {
                                mb_wait(empty + released % S, (released / S) & 1);
                                ++released;
                            }
                            tx += (uint32_t)(wnew - whi) * 8u;
                        } else {
                            wnew = whi;
                        }
                    }
                    slot_rb[slot] = rb;
                    mb_expect(full + slot, tx);
                    unsigned char* st = ring + slot * STB;
                    bulk_g2s(st, gci + cs, (uint32_t)len * (uint32_t)sizeof(Ti), full + slot);
                    bulk_g2s(st + SE * sizeof(Ti), gv + cs, (uint32_t)len * (uint32_t)sizeof(Tv), full + slot);
                    for (int c = whi; c < wnew;) {     // split at the ring wrap and at 32 KB
                        const int sl = c % WCAP;
                        const int cnt = min(min(wnew - c, WCAP - sl), 4096);
                        bulk_g2s(xs + sl, a.x + c, (uint32_t)cnt * 8u, full + slot);
                        c += cnt;
                    }
                    whi = wnew;
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
            const int a0 = eb & ~(kAlign - 1);
            double* P1 = P + (s & 1) * PCAP;
            const int wbase = max(0, rb - a.band) & ~1;     // lowest x row this sub-block reads
            // column -> window slot: slot(col) = (col mod WCAP), via the sub-block's base
            const int cbase = a.slab_base ? __ldg(a.slab_base + (rb >> a.slab_shift)) : 0;
            const int wofs = wbase % WCAP - wbase + cbase;
            if (s >= 2) mb_wait(pempty + (s & 1), ((s >> 1) - 1) & 1);   // sums of sub-block s-2 done
            constexpr int U1 = 4;
            for (int cs = a0; cs < ee; cs += SE, ++it) {
                const int slot = it % S;
                mb_wait(full + slot, (it / S) & 1);
                const Ti* sc = reinterpret_cast<const Ti*>(ring + slot * STB);
                const Tv* sv = reinterpret_cast<const Tv*>(ring + slot * STB + SE * sizeof(Ti));
                const int i0 = max(eb, cs) - cs, i1 = min(ee, cs + SE) - cs;
                for (int ib = i0 + pt; ib < i1; ib += NP * U1) {
                    int sl[U1];
                    double v[U1], px[U1];
#pragma unroll
                    for (int u = 0; u < U1; ++u) {
                        const int i = min(ib + u * NP, i1 - 1);
                        sl[u] = wofs + (int)sc[i];
                        v[u] = (double)sv[i];
                    }
                    compiler_fence();
#pragma unroll
                    for (int u = 0; u < U1; ++u) {
                        if (sl[u] >= WCAP) sl[u] -= WCAP;
                        MRS_DCHECK(sl[u] >= 0 && sl[u] < WCAP);
                        px[u] = xs[sl[u]];
                    }
                    compiler_fence();
#pragma unroll
                    for (int u = 0; u < U1; ++u) {
                        const int i = ib + u * NP;
                        if (i < i1) P1[cs - a0 + i] = mul(v[u], px[u]);
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
    const int mode = a.mode;
    const bool subtract = !(mode == MRS_MODE_ASSIGN || mode == MRS_MODE_ADD);
    const int tid = threadIdx.x;
    int n_lo = __ldg(a.rp + min(R1, R0 + tid)), n_hi = __ldg(a.rp + min(R1, R0 + tid + 1));
    int n_eb = __ldg(a.rp + R0);
    for (int s = 0; s < nsb; ++s) {
        const int rb = R0 + s * T, re = min(R1, rb + T);
        const int row = rb + tid;
        const int lo = n_lo, hi = n_hi, a0 = n_eb & ~(kAlign - 1);
        {
            const int nb = min(R1, rb + T);
            n_eb = __ldg(a.rp + nb);
            n_lo = __ldg(a.rp + min(R1, nb + tid));
            n_hi = __ldg(a.rp + min(R1, nb + tid + 1));
        }
        double acc = 0.0;
        if (row < re) {
            if (mode == MRS_MODE_RSUB) acc = __ldg(a.b + row);
            else if (mode != MRS_MODE_ASSIGN) acc = a.y[row];
        }
        const double* P2 = P + (s & 1) * PCAP;
        mb_wait(pfull + (s & 1), (s >> 1) & 1);
        constexpr int U2 = 4;
        const int klo = lo - a0, khi = hi - a0;
        MRS_DCHECK(klo >= 0 && khi <= PCAP);
        int k = klo;
        if ((k & 1) && k < khi) {                    // odd first product: alone
            const double t = P2[k];
            acc = subtract ? sub(acc, t) : add(acc, t);
            ++k;
        }
        // products as aligned pairs (16-byte shared loads: half the requests of the
        // row-strided, bank-conflicting scalar reads), four per round
        for (; k < khi; k += U2) {
            const int k2 = min(k + 2, ((khi - 1) & ~1));      // second pair (clamped, aligned)
            const double2 p0 = *reinterpret_cast<const double2*>(P2 + k);
            const double2 p1 = *reinterpret_cast<const double2*>(P2 + k2);
            compiler_fence();
            const double t[U2] = {p0.x, p0.y, p1.x, p1.y};
            if (subtract) {
#pragma unroll
                for (int u = 0; u < U2; ++u)
                    if (k + u < khi) acc = sub(acc, t[u]);
            } else {
#pragma unroll
                for (int u = 0; u < U2; ++u)
                    if (k + u < khi) acc = add(acc, t[u]);
            }
        }
        __syncwarp();
        if (tid % 32 == 0) mb_arrive(pempty + (s & 1));
        if (row < re) a.y[row] = acc;
    }
}

template <typename Ti, typename Tv> constexpr int stream_stages() {
    // ring depth by entry size: ~72 KB of entries in flight per SM
    return (int)(sizeof(Ti) + sizeof(Tv)) >= 12 ? 4 : (int)(sizeof(Ti) + sizeof(Tv)) >= 10 ? 5
           : (int)(sizeof(Ti) + sizeof(Tv)) >= 8 ? 6 : 8;
}

int stream_wcap(int band) { return (2 * band + kSumT + 512 + 1) & ~1; }

size_t stream_smem(int band, int entry_bytes, int stages) {
    return (size_t)stream_wcap(band) * 8 + 2 * (size_t)kPcap * 8 + (size_t)stages * kSE * entry_bytes +
           (size_t)(2 * stages + 4) * 8 + (size_t)stages * 4 + 16;
}

template <typename Tv, typename Ti>
cudaError_t stream_launch(const StArgs& a, cudaStream_t s) {
    constexpr int S = stream_stages<Ti, Tv>();
    auto kern = stream_spmv_kernel<Tv, Ti, S>;
    const size_t smem = stream_smem(a.band, (int)(sizeof(Ti) + sizeof(Tv)), S);
    // (per launch: the attribute is per device, and a process may drive several)
    cudaError_t ea = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          227 * 1024);
    if (ea != cudaSuccess) return ea;
    const int nblk = (a.n + kSumT - 1) / kSumT;
    const int grid = std::max(1, std::min(num_sms(), nblk));
    StArgs b = a;
    b.rows_per_cta = ((nblk + grid - 1) / grid) * kSumT;
    kern<<<grid, kSumT + kProdT + 32, smem, s>>>(b);
    return cudaGetLastError();
}

}  // namespace

// The stream variant applies to: one right-hand side, double vectors, plain
// y op= A x (no fused dot / seed / split launch), u16 / slab-u16 / u32 columns,
// a band and a per-256-row entry count that fit shared memory, CSR arrays with 64
// bytes of slack behind them (stages are fetched in 16-byte multiples), 16-byte
// aligned arrays, an even column count (the x window moves in 16-byte pieces).
bool spmm_stream_eligible(const DevCsr& A, int64_t m, const SpArgs& a) {
    if (m != 1 || a.vp != VP_DD || a.dot || a.seed || a.row0 || a.vrows || a.guard) return false;
    if (!A.padded || A.band < 0 || A.blk_max <= 0) return false;
    if (A.ib != 2 && A.ib != 4) return false;
    if (A.vb != 4 && A.vb != 8) return false;
    if (A.nrows < 1 || A.nnz < 1 || (A.ncols & 1)) return false;
    if (A.blk_max + kAlign > kPcap) return false;
    if (A.slab_base && (A.slab_shift < 8)) return false;      // a 256-row sub-block in one slab
    const int S = A.ib + A.vb >= 12 ? 4 : A.ib + A.vb >= 10 ? 5 : A.ib + A.vb >= 8 ? 6 : 8;
    if (stream_smem(A.band, A.ib + A.vb, S) > 227 * 1024) return false;
    auto al16 = [](const void* p) { return ((uintptr_t)p & 15u) == 0; };
    return al16(A.ci) && al16(A.v) && al16(a.x);
}

static std::atomic<int64_t> g_stream_launches{0};
int64_t spmm_stream_launches() { return g_stream_launches.load(); }

cudaError_t launch_spmm_stream(const DevCsr& A, const SpArgs& a, cudaStream_t s) {
    g_stream_launches.fetch_add(1);
    StArgs t;
    t.rp = A.rp; t.ci = A.ci; t.vals = A.v;
    t.slab_base = A.slab_base; t.slab_shift = A.slab_shift;
    t.x = a.x; t.b = a.b; t.y = a.y;
    t.n = (int)A.nrows; t.ncols = (int)A.ncols; t.band = A.band;
    t.rows_per_cta = 0; t.wcap = stream_wcap(A.band); t.mode = a.mode;
    if (A.vb == 8) return A.ib == 4 ? stream_launch<double, uint32_t>(t, s)
                                    : stream_launch<double, uint16_t>(t, s);
    return A.ib == 4 ? stream_launch<float, uint32_t>(t, s) : stream_launch<float, uint16_t>(t, s);
}

}  // namespace mrs
