// spmm_probe.cu -- standalone A/B of SpMM kernel designs (not part of the
// library).  Builds the bench matrices on the host, runs each variant after an
// L2 flush, checks every variant bitwise against the first, prints us/launch
// and algorithmic GB/s.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
//        -o spmm_probe spmm_probe.cu && ./spmm_probe
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
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ void fence() { asm volatile("" ::: "memory"); }

template <int M> struct Lay {
    static constexpr int CPL = (M == 1) ? 1 : 2;
    static constexpr int LPR = M / CPL;
};

struct Args {
    const int* rp;
    const void* ci;
    const double* v;
    const int* slab;   // null: absolute columns
    int slab_shift;
    int n;
    const double* x;
    const double* b;
    double* y;
    int chunk;
    int tiles;         // tma: number of tiles
    int tile_rows;
    int tiles_per_chunk;
    const int* sptr;          // sell: slice entry offsets
    const uint8_t* slen;      // sell: row lengths
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

// ---------------------------------------------------------------- baseline
// replica of the library's spmm_kernel<M, OP_SPMV RSUB>: lanes over columns,
// groups of UNR entries, chunk-strided one-wave grid.
template <int M, typename Ti, int UNR, int MINB, int OWN = 0>
__global__ void __launch_bounds__(256, MINB) k_base(Args a) {
    constexpr int CPL = Lay<M>::CPL, LPR = Lay<M>::LPR, RPB = 256 / LPR;
    const int cofs = (threadIdx.x % LPR) * CPL;
    const Ti* ci = (const Ti*)a.ci;
    for (int r0 = blockIdx.x * a.chunk; r0 < a.n; r0 += gridDim.x * a.chunk) {
        const int r1 = min(r0 + a.chunk, a.n);
        for (int row = r0 + threadIdx.x / LPR; row < r1; row += RPB) {
            const int base = a.slab ? __ldg(a.slab + (row >> a.slab_shift)) : 0;
            const int lo = __ldg(a.rp + row), hi = __ldg(a.rp + row + 1);
            const int o = row * M + cofs;
            V<CPL> acc = ldx<CPL>(a.b + o);
            for (int k = lo; k < hi; k += UNR) {
                int c[UNR]; double v[UNR]; V<CPL> g[UNR];
#pragma unroll
                for (int u = 0; u < UNR; ++u) {
                    const int kk = (k + u < hi) ? k + u : lo;
                    c[u] = base + (int)__ldg(ci + kk);
                    v[u] = __ldg(a.v + kk);
                }
                fence();
                if (OWN == 1) {
#pragma unroll
                    for (int u = 0; u < UNR; ++u) c[u] = (c[u] & 0) + row;   // keep the dependency, hit own row
                }
#pragma unroll
                for (int u = 0; u < UNR; ++u) g[u] = ldx<CPL>(a.x + c[u] * M + cofs);
                fence();
#pragma unroll
                for (int u = 0; u < UNR; ++u)
                    if (k + u < hi)
#pragma unroll
                        for (int i = 0; i < CPL; ++i) acc.v[i] = sub(acc.v[i], mul(v[u], g[u].v[i]));
            }
            stv<CPL>(a.y + o, acc);
        }
    }
}

// ---------------------------------------------------------------- TMA staged
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

// Stage layout (bytes): rp [RPS] ints | ci [EC] Ti | v [EC] doubles | b [T*M] doubles
template <int M, typename Ti, int NCW, int S, int EPR>
struct TmaCfg {
    static constexpr int CPL = Lay<M>::CPL, LPR = Lay<M>::LPR;
    static constexpr int T = NCW * 32 / LPR;               // rows per tile (stage)
    static constexpr int RPS = ((T + 1 + 3) / 4 + 1) * 4;  // rp slots (aligned superset)
    static constexpr int EC = EPR * T + 16;                // entry capacity
    static constexpr int RP_B = RPS * 4;
    static constexpr int CI_B = ((EC * (int)sizeof(Ti) + 15) / 16) * 16;
    static constexpr int V_B = EC * 8;
    static constexpr int B_B = T * M * 8;
    static constexpr int STAGE = RP_B + CI_B + V_B + B_B;
    static constexpr int SMEM = S * STAGE + 2 * S * 8;
};

template <int M, typename Ti, int NCW, int S, int EPR, int UNR>
__global__ void __launch_bounds__((NCW + 1) * 32, 1) k_tma(Args a) {
    using C = TmaCfg<M, Ti, NCW, S, EPR>;
    constexpr int CPL = C::CPL, LPR = C::LPR, T = C::T;
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + S * C::STAGE);
    uint64_t* empty = full + S;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) { mb_init(full + s, 1); mb_init(empty + s, NCW); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // this CTA's tiles: chunks of tiles_per_chunk consecutive tiles, strided over the grid
    const int tpc = a.tiles_per_chunk;
    const int nchunks = (a.tiles + tpc - 1) / tpc;
    if (warp == NCW) {   // producer: tile extents for 32 iterations per round trip
        for (int it0 = 0;; it0 += 32) {
            const int itj = it0 + lane;
            const int chj = blockIdx.x + (itj / tpc) * gridDim.x;
            const int tj = chj * tpc + itj % tpc;
            const bool vj = chj < nchunks && tj < a.tiles;
            int e0j = 0, e1j = 0;
            if (vj) {
                const int r0 = tj * T, r1 = min(r0 + T, a.n);
                e0j = __ldg(a.rp + r0);
                e1j = __ldg(a.rp + r1);
            }
            const unsigned vmask = __ballot_sync(~0u, vj);
            if (!vmask) break;
            for (int j = 0; j < 32 && ((vmask >> j) & 1); ++j) {
                const int e0 = __shfl_sync(~0u, e0j, j), e1 = __shfl_sync(~0u, e1j, j);
                const int t = __shfl_sync(~0u, tj, j);
                const int it = it0 + j;
                if (lane == 0) {
                    const int s = it % S;
                    if (it >= S) mb_wait(empty + s, ((it / S) & 1) ^ 1);
                    unsigned char* st = sm + s * C::STAGE;
                    const int r0 = t * T, r1 = min(r0 + T, a.n);
                    const int ra = r0 & ~3, rb = (r1 + 1 + 3) & ~3;
                    constexpr int EA = 16 / (int)sizeof(Ti);
                    const int ca = e0 & ~(EA - 1), cb = (e1 + EA - 1) & ~(EA - 1);
                    const int va = e0 & ~1, vb = (e1 + 1) & ~1;
                    const bool fits = (cb - ca) <= C::EC && (vb - va) <= C::EC;
                    const uint32_t bb = ((r1 - r0) * M * 8 + 15) & ~15u;
                    uint32_t bytes = (rb - ra) * 4 + bb;
                    if (fits) bytes += (cb - ca) * sizeof(Ti) + (vb - va) * 8;
                    mb_expect(full + s, bytes);
                    bulk_g2s(st, a.rp + ra, (rb - ra) * 4, full + s);
                    if (fits) {
                        bulk_g2s(st + C::RP_B, (const Ti*)a.ci + ca, (cb - ca) * sizeof(Ti), full + s);
                        bulk_g2s(st + C::RP_B + C::CI_B, a.v + va, (vb - va) * 8, full + s);
                    }
                    bulk_g2s(st + C::RP_B + C::CI_B + C::V_B, a.b + (size_t)r0 * M, bb, full + s);
                }
                __syncwarp();
            }
        }
        return;
    }
    // consumers
    const int cofs = (lane % LPR) * CPL;
    const int rit = warp * (32 / LPR) + lane / LPR;   // row within tile
    const Ti* gci = (const Ti*)a.ci;
    int it = 0;
    for (int ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
        const int t1 = min((ch + 1) * tpc, a.tiles);
        for (int t = ch * tpc; t < t1; ++t, ++it) {
            const int s = it % S;
            mb_wait(full + s, (it / S) & 1);
            const unsigned char* st = sm + s * C::STAGE;
            const int* srp = reinterpret_cast<const int*>(st);
            const Ti* sci = reinterpret_cast<const Ti*>(st + C::RP_B);
            const double* sv = reinterpret_cast<const double*>(st + C::RP_B + C::CI_B);
            const double* sb = reinterpret_cast<const double*>(st + C::RP_B + C::CI_B + C::V_B);
            const int r0 = t * T;
            const int row = r0 + rit;
            if (row < a.n) {
                const int ra = r0 & ~3;
                const int e0 = srp[r0 - ra];
                const int r1 = min(r0 + T, a.n);
                const int e1 = srp[r1 - ra];
                constexpr int EA = 16 / (int)sizeof(Ti);
                const int ca = e0 & ~(EA - 1), cb = (e1 + EA - 1) & ~(EA - 1);
                const int va = e0 & ~1, vb = (e1 + 1) & ~1;
                const bool fits = (cb - ca) <= C::EC && (vb - va) <= C::EC;
                const int lo = srp[row - ra], hi = srp[row + 1 - ra];
                const int base = a.slab ? __ldg(a.slab + (row >> a.slab_shift)) : 0;
                V<CPL> acc;
#pragma unroll
                for (int i = 0; i < CPL; ++i) acc.v[i] = sb[rit * M + cofs + i];
                for (int k = lo; k < hi; k += UNR) {
                    V<CPL> g[UNR];
                    int c[UNR];
#pragma unroll
                    for (int u = 0; u < UNR; ++u) {
                        const int kk = (k + u < hi) ? k + u : lo;
                        c[u] = base + (int)(fits ? sci[kk - ca] : __ldg(gci + kk));
                    }
#pragma unroll
                    for (int u = 0; u < UNR; ++u) g[u] = ldx<CPL>(a.x + c[u] * M + cofs);
                    fence();
#pragma unroll
                    for (int u = 0; u < UNR; ++u)
                        if (k + u < hi) {
                            const double vv = fits ? sv[k + u - va] : __ldg(a.v + k + u);
#pragma unroll
                            for (int i = 0; i < CPL; ++i) acc.v[i] = sub(acc.v[i], mul(vv, g[u].v[i]));
                        }
                }
                stv<CPL>(a.y + (size_t)row * M + cofs, acc);
            }
            __syncwarp();
            if (lane == 0) mb_arrive(empty + s);
        }
    }
}


// ---------------------------------------------------------------- matrices
struct Csr {
    std::string name;
    int n;
    std::vector<int> rp;
    std::vector<uint32_t> ci;
    std::vector<double> v;
};

static Csr poisson7(int g) {
    Csr A;
    A.name = "7pt-" + std::to_string(g);
    A.n = g * g * g;
    A.rp.push_back(0);
    std::mt19937_64 rng(1);
    std::uniform_real_distribution<double> U(-1, 1);
    for (int z = 0; z < g; ++z)
        for (int y = 0; y < g; ++y)
            for (int x = 0; x < g; ++x) {
                const int i = (z * g + y) * g + x;
                auto add = [&](int j) { A.ci.push_back(j); A.v.push_back(j == i ? 6.0 + U(rng) : U(rng)); };
                if (z > 0) add(i - g * g);
                if (y > 0) add(i - g);
                if (x > 0) add(i - 1);
                add(i);
                if (x < g - 1) add(i + 1);
                if (y < g - 1) add(i + g);
                if (z < g - 1) add(i + g * g);
                A.rp.push_back((int)A.ci.size());
            }
    return A;
}


static Csr stencil27(int g) {
    Csr A;
    A.name = "27pt-" + std::to_string(g);
    A.n = g * g * g;
    A.rp.push_back(0);
    std::mt19937_64 rng(4);
    std::uniform_real_distribution<double> U(-1, 1);
    for (int z = 0; z < g; ++z)
        for (int y = 0; y < g; ++y)
            for (int x = 0; x < g; ++x) {
                const int i = (z * g + y) * g + x;
                for (int dz = -1; dz <= 1; ++dz)
                    for (int dy = -1; dy <= 1; ++dy)
                        for (int dx = -1; dx <= 1; ++dx) {
                            const int zz = z + dz, yy = y + dy, xx = x + dx;
                            if (zz < 0 || yy < 0 || xx < 0 || zz >= g || yy >= g || xx >= g) continue;
                            const int j = (zz * g + yy) * g + xx;
                            A.ci.push_back(j);
                            A.v.push_back(j == i ? 30.0 + U(rng) : U(rng));
                        }
                A.rp.push_back((int)A.ci.size());
            }
    return A;
}

static Csr band_random(int n, int band, double mean) {
    Csr A;
    A.name = "c5-" + std::to_string(n);
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

// slab compression: 2^s rows per slab, base = min column of the slab; largest s fitting 16 bits
static bool slab_compress(const Csr& A, int& shift, std::vector<int>& base, std::vector<uint16_t>& c16) {
    for (shift = 24; shift >= 6; --shift) {
        const int ns = (A.n + (1 << shift) - 1) >> shift;
        base.assign(ns, 0);
        bool ok = true;
        for (int s = 0; s < ns && ok; ++s) {
            const int r0 = s << shift, r1 = std::min(A.n, (s + 1) << shift);
            uint32_t mn = UINT32_MAX, mx = 0;
            for (int k = A.rp[r0]; k < A.rp[r1]; ++k) { mn = std::min(mn, A.ci[k]); mx = std::max(mx, A.ci[k]); }
            if (mn == UINT32_MAX) mn = 0;
            if (mx - mn >= 65536) ok = false;
            base[s] = (int)mn;
        }
        if (!ok) continue;
        c16.resize(A.ci.size());
        for (int r = 0; r < A.n; ++r)
            for (int k = A.rp[r]; k < A.rp[r + 1]; ++k) c16[k] = (uint16_t)(A.ci[k] - base[r >> shift]);
        return true;
    }
    return false;
}

template <typename T> static T* up(const std::vector<T>& h, size_t pad = 64) {
    T* d;
    CK(cudaMalloc(&d, (h.size() + pad) * sizeof(T)));
    CK(cudaMemset(d, 0, (h.size() + pad) * sizeof(T)));
    CK(cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
    return d;
}

static double* g_flush;
static int g_chunk_rows = 0;
static void flush_l2() {
    CK(cudaMemsetAsync(g_flush, 0, 256u << 20));
}

template <class F> static float time_b2b_us(F&& f, int reps = 40) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    f();
    flush_l2();
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) f();
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms * 1e3f / reps;
}
template <class F> static float time_us(F&& f, int reps = 15) {
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

template <int M, typename Ti, int UNR, int MINB, int OWN = 0>
static void run_base(Args a, int& grid) {
    auto kern = k_base<M, Ti, UNR, MINB, OWN>;
    int bps;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, 256, 0);
    constexpr int RPB = 256 / Lay<M>::LPR;
    const long cap = (long)bps * nsm();
    const long P = (a.n + RPB - 1) / RPB, ppc = (P + cap - 1) / cap;
    long pmax = RPB >= 512 ? 1 : 512 / RPB;
    if (g_chunk_rows) pmax = std::max(1, g_chunk_rows / RPB);
    const long sp = std::min(ppc, pmax);
    const long nch = (P + sp - 1) / sp, cpc = (nch + cap - 1) / cap;
    grid = (int)((nch + cpc - 1) / cpc);
    a.chunk = (int)(RPB * sp);
    kern<<<grid, 256>>>(a);
}

template <int M, typename Ti, int NCW, int S, int EPR, int UNR>
static void run_tma(Args a, int tpc_override, int ctas_per_sm) {
    using C = TmaCfg<M, Ti, NCW, S, EPR>;
    auto kern = k_tma<M, Ti, NCW, S, EPR, UNR>;
    static bool set = false;
    if (!set) { CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM)); set = true; }
    int bps;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, (NCW + 1) * 32, C::SMEM);
    if (ctas_per_sm > 0 && ctas_per_sm < bps) bps = ctas_per_sm;
    a.tile_rows = C::T;
    a.tiles = (a.n + C::T - 1) / C::T;
    const long cap = (long)bps * nsm();
    const long tpcta = (a.tiles + cap - 1) / cap;
    long tpc = tpc_override > 0 ? tpc_override : std::min<long>(tpcta, std::max(1, 512 / C::T));
    a.tiles_per_chunk = (int)tpc;
    const long nch = (a.tiles + tpc - 1) / tpc;
    const long cpc = (nch + cap - 1) / cap;
    const int grid = (int)((nch + cpc - 1) / cpc);
    kern<<<grid, (NCW + 1) * 32, C::SMEM>>>(a);
}


// ---------------------------------------------------------------- SELL-C
// Slices of C = 32/LPR consecutive rows (one warp's rows); entry k of row r
// lives at sptr[r/C] + k*C + r%C (slice padded to its longest row), so a
// warp's load of entry k for its C rows is one contiguous segment.
template <int M, typename Ti, int UNR, int MINB>
__global__ void __launch_bounds__(256, MINB) k_sell(Args a) {
    constexpr int CPL = Lay<M>::CPL, LPR = Lay<M>::LPR, RPB = 256 / LPR, C = 32 / LPR;
    const int cofs = (threadIdx.x % LPR) * CPL;
    const Ti* ci = (const Ti*)a.ci;
    for (int r0 = blockIdx.x * a.chunk; r0 < a.n; r0 += gridDim.x * a.chunk) {
        const int r1 = min(r0 + a.chunk, a.n);
        for (int row = r0 + threadIdx.x / LPR; row < r1; row += RPB) {
            const int base = a.slab ? __ldg(a.slab + (row >> a.slab_shift)) : 0;
            const int p = __ldg(a.sptr + row / C) + row % C;
            const int len = __ldg(a.slen + row);
            const int o = row * M + cofs;
            V<CPL> acc = ldx<CPL>(a.b + o);
            for (int k = 0; k < len; k += UNR) {
                int c[UNR]; double v[UNR]; V<CPL> g[UNR];
#pragma unroll
                for (int u = 0; u < UNR; ++u) {
                    const int kk = (k + u < len) ? k + u : 0;
                    c[u] = base + (int)__ldg(ci + p + kk * C);
                    v[u] = __ldg(a.v + p + kk * C);
                }
                fence();
#pragma unroll
                for (int u = 0; u < UNR; ++u) g[u] = ldx<CPL>(a.x + c[u] * M + cofs);
                fence();
#pragma unroll
                for (int u = 0; u < UNR; ++u)
                    if (k + u < len)
#pragma unroll
                        for (int i = 0; i < CPL; ++i) acc.v[i] = sub(acc.v[i], mul(v[u], g[u].v[i]));
            }
            stv<CPL>(a.y + o, acc);
        }
    }
}

template <int M, typename Ti, int UNR, int MINB>
static void run_sell(Args a) {
    auto kern = k_sell<M, Ti, UNR, MINB>;
    int bps;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, 256, 0);
    constexpr int RPB = 256 / Lay<M>::LPR;
    const long cap = (long)bps * nsm();
    const long P = (a.n + RPB - 1) / RPB, ppc = (P + cap - 1) / cap;
    const long pmax = RPB >= 512 ? 1 : 512 / RPB, sp = std::min(ppc, pmax);
    const long nch = (P + sp - 1) / sp, cpc = (nch + cap - 1) / cap;
    const int grid = (int)((nch + cpc - 1) / cpc);
    a.chunk = (int)(RPB * sp);
    kern<<<grid, 256>>>(a);
}

// host: SELL-C arrays from CSR (indices given as Ti array matching A's entries)
template <typename Ti>
static void to_sell(const Csr& A, const std::vector<Ti>& cols, int C, std::vector<int>& sptr,
                    std::vector<uint8_t>& slen, std::vector<Ti>& sci, std::vector<double>& sv) {
    const int ns = (A.n + C - 1) / C;
    sptr.assign(ns + 1, 0);
    slen.assign(A.n, 0);
    long tot = 0;
    for (int s = 0; s < ns; ++s) {
        int L = 0;
        for (int r = s * C; r < std::min(A.n, s * C + C); ++r) {
            const int l = A.rp[r + 1] - A.rp[r];
            slen[r] = (uint8_t)l;
            L = std::max(L, l);
        }
        sptr[s] = (int)tot;
        tot += (long)L * C;
    }
    sptr[ns] = (int)tot;
    sci.assign(tot, 0);
    sv.assign(tot, 0.0);
    for (int r = 0; r < A.n; ++r) {
        const int s = r / C, L = (sptr[s + 1] - sptr[s]) / C;
        const int lo = A.rp[r], l = A.rp[r + 1] - lo;
        for (int k = 0; k < L; ++k) {
            const int kk = k < l ? k : 0;
            sci[sptr[s] + k * C + r % C] = l ? cols[lo + kk] : 0;
            sv[sptr[s] + k * C + r % C] = k < l ? A.v[lo + k] : 0.0;
        }
    }
}



// base + cross-pass register prefetch: the next pass's row pointers (PF>=1)
// and its first entry group's columns/values (PF>=2) are loaded while the
// current row is accumulated.
template <int M, typename Ti, int UNR, int MINB, int PF>
__global__ void __launch_bounds__(256, MINB) k_pf(Args a) {
    constexpr int CPL = Lay<M>::CPL, LPR = Lay<M>::LPR, RPB = 256 / LPR;
    const int cofs = (threadIdx.x % LPR) * CPL;
    const Ti* ci = (const Ti*)a.ci;
    // flattened (chunk, pass) iteration for this thread
    int r0 = blockIdx.x * a.chunk;
    int row = r0 + threadIdx.x / LPR;
    auto advance = [&](int& c0, int& rw) {
        rw += RPB;
        if (rw >= min(c0 + a.chunk, a.n)) { c0 += gridDim.x * a.chunk; rw = c0 + threadIdx.x / LPR; }
    };
    // skip rows past a short chunk end
    while (r0 < a.n && row >= min(r0 + a.chunk, a.n)) { r0 += gridDim.x * a.chunk; row = r0 + threadIdx.x / LPR; }
    if (r0 >= a.n) return;
    int lo = __ldg(a.rp + row), hi = __ldg(a.rp + row + 1);
    int pc[UNR]; double pv[UNR];
    if constexpr (PF >= 2) {
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const int kk = (lo + u < hi) ? lo + u : lo;
            pc[u] = (int)__ldg(ci + kk); pv[u] = __ldg(a.v + kk);
        }
    }
    while (true) {
        int nr0 = r0, nrow = row;
        advance(nr0, nrow);
        const bool more = nr0 < a.n && nrow < a.n;
        int nlo = 0, nhi = 0;
        if (more) { nlo = __ldg(a.rp + nrow); nhi = __ldg(a.rp + nrow + 1); }
        const int base = a.slab ? __ldg(a.slab + (row >> a.slab_shift)) : 0;
        const int o = row * M + cofs;
        V<CPL> acc = ldx<CPL>(a.b + o);
        for (int k = lo; k < hi; k += UNR) {
            int c[UNR]; double v[UNR]; V<CPL> g[UNR];
            if (PF >= 2 && k == lo) {
#pragma unroll
                for (int u = 0; u < UNR; ++u) { c[u] = base + pc[u]; v[u] = pv[u]; }
            } else {
#pragma unroll
                for (int u = 0; u < UNR; ++u) {
                    const int kk = (k + u < hi) ? k + u : lo;
                    c[u] = base + (int)__ldg(ci + kk);
                    v[u] = __ldg(a.v + kk);
                }
            }
            fence();
#pragma unroll
            for (int u = 0; u < UNR; ++u) g[u] = ldx<CPL>(a.x + c[u] * M + cofs);
            fence();
#pragma unroll
            for (int u = 0; u < UNR; ++u)
                if (k + u < hi)
#pragma unroll
                    for (int i = 0; i < CPL; ++i) acc.v[i] = sub(acc.v[i], mul(v[u], g[u].v[i]));
        }
        stv<CPL>(a.y + o, acc);
        if (!more) break;
        r0 = nr0; row = nrow; lo = nlo; hi = nhi;
        if constexpr (PF >= 2) {
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                const int kk = (lo + u < hi) ? lo + u : lo;
                pc[u] = (int)__ldg(ci + kk); pv[u] = __ldg(a.v + kk);
            }
        }
    }
}

template <int M, typename Ti, int UNR, int MINB, int PF>
static void run_pf(Args a) {
    auto kern = k_pf<M, Ti, UNR, MINB, PF>;
    int bps;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, 256, 0);
    constexpr int RPB = 256 / Lay<M>::LPR;
    const long cap = (long)bps * nsm();
    const long P = (a.n + RPB - 1) / RPB, ppc = (P + cap - 1) / cap;
    long pmax = std::max(1, 64 / RPB);
    const long sp = std::min(ppc, pmax);
    const long nch = (P + sp - 1) / sp, cpc = (nch + cap - 1) / cap;
    const int grid = (int)((nch + cpc - 1) / cpc);
    a.chunk = (int)(RPB * sp);
    kern<<<grid, 256>>>(a);
}


// ---------------------------------------------------------------- SELL-4
// Slices of C = 32/LPR rows; within a slice, entries are grouped by 4:
// group g of row r (entries 4g..4g+3) is stored contiguously at
// sptr[slice] + g*4*C + (r%C)*4.  Rows padded to the slice's group count.
// A lane loads its row's whole group with one 32-byte (values) and one
// 8/16-byte (columns) access; a warp instruction covers C rows' groups =
// one contiguous 4*C-entry block.
__device__ __forceinline__ void ld4(const double* p, double (&v)[4]) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(p));
    const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
}
template <typename Ti> struct Grp;
template <> struct Grp<uint16_t> {
    static __device__ __forceinline__ void ld(const uint16_t* p, int (&c)[4]) {
        uint2 t = __ldg(reinterpret_cast<const uint2*>(p));
        c[0] = t.x & 0xffff; c[1] = t.x >> 16; c[2] = t.y & 0xffff; c[3] = t.y >> 16;
    }
};
template <> struct Grp<uint32_t> {
    static __device__ __forceinline__ void ld(const uint32_t* p, int (&c)[4]) {
        uint4 t = __ldg(reinterpret_cast<const uint4*>(p));
        c[0] = t.x; c[1] = t.y; c[2] = t.z; c[3] = t.w;
    }
};

template <int M, typename Ti, int MINB, int PIPE>
__global__ void __launch_bounds__(256, MINB) k_g4(Args a) {
    constexpr int CPL = Lay<M>::CPL, LPR = Lay<M>::LPR, RPB = 256 / LPR, C = 32 / LPR;
    const int cofs = (threadIdx.x % LPR) * CPL;
    const Ti* ci = (const Ti*)a.ci;
    for (int r0 = blockIdx.x * a.chunk; r0 < a.n; r0 += gridDim.x * a.chunk) {
        const int r1 = min(r0 + a.chunk, a.n);
        for (int row = r0 + threadIdx.x / LPR; row < r1; row += RPB) {
            const int base = a.slab ? __ldg(a.slab + (row >> a.slab_shift)) : 0;
            const int p = __ldg(a.sptr + row / C) + (row % C) * 4;
            const int len = __ldg(a.slen + row);
            const int o = row * M + cofs;
            V<CPL> acc = ldx<CPL>(a.b + o);
            int c[4]; double v[4];
            if (len > 0) {
                Grp<Ti>::ld(ci + p, c);
                ld4(a.v + p, v);
            }
            for (int k = 0; k < len; k += 4) {
                V<CPL> g[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) g[u] = ldx<CPL>(a.x + (base + c[u]) * M + cofs);
                double w[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) w[u] = v[u];
                if (PIPE && k + 4 < len) {   // next group's entries fly with this group's gathers
                    const int q = p + (k + 4) * C;
                    Grp<Ti>::ld(ci + q, c);
                    ld4(a.v + q, v);
                }
                fence();
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (k + u < len)
#pragma unroll
                        for (int i = 0; i < CPL; ++i) acc.v[i] = sub(acc.v[i], mul(w[u], g[u].v[i]));
                if (!PIPE && k + 4 < len) {
                    const int q = p + (k + 4) * C;
                    Grp<Ti>::ld(ci + q, c);
                    ld4(a.v + q, v);
                }
            }
            stv<CPL>(a.y + o, acc);
        }
    }
}

template <int M, typename Ti, int MINB, int PIPE>
static void run_g4(Args a) {
    auto kern = k_g4<M, Ti, MINB, PIPE>;
    int bps;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, 256, 0);
    constexpr int RPB = 256 / Lay<M>::LPR;
    const long cap = (long)bps * nsm();
    const long P = (a.n + RPB - 1) / RPB, ppc = (P + cap - 1) / cap;
    long pmax = std::max(1, 64 / RPB);
    const long sp = std::min(ppc, pmax);
    const long nch = (P + sp - 1) / sp, cpc = (nch + cap - 1) / cap;
    const int grid = (int)((nch + cpc - 1) / cpc);
    a.chunk = (int)(RPB * sp);
    kern<<<grid, 256>>>(a);
}

template <typename Ti>
static void to_g4(const Csr& A, const std::vector<Ti>& cols, int C, std::vector<int>& sptr,
                  std::vector<uint8_t>& slen, std::vector<Ti>& sci, std::vector<double>& sv) {
    const int ns = (A.n + C - 1) / C;
    sptr.assign(ns + 1, 0);
    slen.assign(A.n, 0);
    long tot = 0;
    for (int s = 0; s < ns; ++s) {
        int G = 0;
        for (int r = s * C; r < std::min(A.n, s * C + C); ++r) {
            const int l = A.rp[r + 1] - A.rp[r];
            slen[r] = (uint8_t)l;
            G = std::max(G, (l + 3) / 4);
        }
        sptr[s] = (int)tot;
        tot += (long)G * 4 * C;
    }
    sptr[ns] = (int)tot;
    sci.assign(tot, 0);
    sv.assign(tot, 0.0);
    for (int r = 0; r < A.n; ++r) {
        const int s = r / C, G = (sptr[s + 1] - sptr[s]) / (4 * C);
        const int lo = A.rp[r], l = A.rp[r + 1] - lo;
        for (int k = 0; k < 4 * G; ++k) {
            const long q = sptr[s] + (long)(k / 4) * 4 * C + (r % C) * 4 + k % 4;
            sci[q] = l ? cols[lo + (k < l ? k : 0)] : 0;
            sv[q] = k < l ? A.v[lo + k] : 0.0;
        }
    }
}


// cooperative entry loads: the LPR lanes of a row load LPR consecutive
// entries (one each) and exchange them by shuffles, instead of every lane
// loading every entry.  Warp-uniform trip count (max row length in the warp).
template <int M, typename Ti, int MINB, int G2 = 1>
__global__ void __launch_bounds__(256, MINB) k_coop(Args a) {
    constexpr int CPL = Lay<M>::CPL, LPR = Lay<M>::LPR, RPB = 256 / LPR;
    constexpr int G = LPR * G2;                 // entries per group
    const int l = threadIdx.x % LPR;
    const int cofs = l * CPL;
    const int gbase = (threadIdx.x % 32) & ~(LPR - 1);
    const Ti* ci = (const Ti*)a.ci;
    for (int r0 = blockIdx.x * a.chunk; r0 < a.n; r0 += gridDim.x * a.chunk) {
        const int r1 = min(r0 + a.chunk, a.n);
        for (int rb = r0; rb < r1; rb += RPB) {        // warp-uniform pass loop
            const int row = rb + threadIdx.x / LPR;
            const bool live = row < r1;
            const int base = (live && a.slab) ? __ldg(a.slab + (row >> a.slab_shift)) : 0;
            const int lo = live ? __ldg(a.rp + row) : 0, hi = live ? __ldg(a.rp + row + 1) : 0;
            const int len = hi - lo;
            const int wlen = __reduce_max_sync(0xffffffffu, len);
            const int o = row * M + cofs;
            V<CPL> acc;
            if (live) acc = ldx<CPL>(a.b + o);
            for (int k = 0; k < wlen; k += G) {
                int cm[G2]; double vm[G2];
#pragma unroll
                for (int j = 0; j < G2; ++j) {
                    const int e = k + j * LPR + l;
                    const int kk = e < len ? lo + e : lo;
                    cm[j] = (len > 0) ? base + (int)__ldg(ci + kk) : 0;
                    vm[j] = (len > 0) ? __ldg(a.v + kk) : 0.0;
                }
                V<CPL> g[G];
                const bool act = live && k < len;
#pragma unroll
                for (int j = 0; j < G2; ++j)
#pragma unroll
                    for (int u = 0; u < LPR; ++u) {
                        const int cu = __shfl_sync(0xffffffffu, cm[j], gbase + u);
                        if (act) g[j * LPR + u] = ldx<CPL>(a.x + cu * M + cofs);
                    }
                fence();
#pragma unroll
                for (int j = 0; j < G2; ++j)
#pragma unroll
                    for (int u = 0; u < LPR; ++u) {
                        const double vu = __shfl_sync(0xffffffffu, vm[j], gbase + u);
                        if (act && k + j * LPR + u < len)
#pragma unroll
                            for (int i = 0; i < CPL; ++i)
                                acc.v[i] = sub(acc.v[i], mul(vu, g[j * LPR + u].v[i]));
                    }
            }
            if (live) stv<CPL>(a.y + o, acc);
        }
    }
}

template <int M, typename Ti, int MINB, int G2>
static void run_coop(Args a) {
    auto kern = k_coop<M, Ti, MINB, G2>;
    int bps;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, 256, 0);
    constexpr int RPB = 256 / Lay<M>::LPR;
    const long cap = (long)bps * nsm();
    const long P = (a.n + RPB - 1) / RPB, ppc = (P + cap - 1) / cap;
    long pmax = std::max(1, 64 / RPB);
    const long sp = std::min(ppc, pmax);
    const long nch = (P + sp - 1) / sp, cpc = (nch + cap - 1) / cap;
    const int grid = (int)((nch + cpc - 1) / cpc);
    a.chunk = (int)(RPB * sp);
    kern<<<grid, 256>>>(a);
}

static double bytes_of(const Csr& A, int m, int ib, int nslab) {
    return (double)A.ci.size() * (8 + ib) + (A.n + 1) * 4.0 + nslab * 4.0 + 3.0 * A.n * m * 8;
}

template <int M, typename Ti, int NCW, int S, int EPR, int UNR>
static float try_tma(Args a, int tpc, int cps) {
    if constexpr (TmaCfg<M, Ti, NCW, S, EPR>::SMEM > 227 * 1024) return -1.f;
    else return time_us([&] { run_tma<M, Ti, NCW, S, EPR, UNR>(a, tpc, cps); });
}

template <int M, int EPR> static void bench_matrix(const Csr& A) {
    if (getenv("ONLY_M") && atoi(getenv("ONLY_M")) != M) return;
    std::vector<double> hx((size_t)A.n * M), hb((size_t)A.n * M);
    std::mt19937_64 rng(7);
    std::uniform_real_distribution<double> U(-1, 1);
    for (auto& t : hx) t = U(rng);
    for (auto& t : hb) t = U(rng);
    double* x = up(hx, 64 * M);
    double* b = up(hb, 64 * M);
    double *y0, *y1;
    CK(cudaMalloc(&y0, hx.size() * 8 + 4096));
    CK(cudaMalloc(&y1, hx.size() * 8 + 4096));
    int* rp = up(A.rp);
    uint32_t* ci32 = up(A.ci);
    double* v = up(A.v);
    int shift;
    std::vector<int> hbase;
    std::vector<uint16_t> c16;
    const bool slab = slab_compress(A, shift, hbase, c16);
    uint16_t* ci16 = slab ? up(c16, 128) : nullptr;
    int* sb = slab ? up(hbase) : nullptr;
    std::vector<double> ref((size_t)A.n * M), out((size_t)A.n * M);

    auto check = [&](const char* name, double us, double byts) {
        CK(cudaMemcpy(out.data(), y1, out.size() * 8, cudaMemcpyDeviceToHost));
        const bool eq = memcmp(out.data(), ref.data(), out.size() * 8) == 0;
        printf("  %-40s %9.2f us  %6.0f GB/s  %s\n", name, us, byts / us / 1e3, eq ? "bitwise" : "MISMATCH");
        CK(cudaMemset(y1, 0, out.size() * 8));
    };
    printf("%s n=%d nnz=%zu m=%d slab=%d(shift %d)\n", A.name.c_str(), A.n, A.ci.size(), M, (int)slab, shift);
    Args a{};
    a.rp = rp; a.v = v; a.n = A.n; a.x = x; a.b = b;
    // reference output: base u32
    {
        Args r = a; r.ci = ci32; r.y = y0; int g;
        run_base<M, uint32_t, 4, 6>(r, g);
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(ref.data(), y0, ref.size() * 8, cudaMemcpyDeviceToHost));
    }
    const double b32 = bytes_of(A, M, 4, 0);
    const double b16 = slab ? bytes_of(A, M, 2, (int)hbase.size()) : 0;
    Args a32 = a; a32.ci = ci32; a32.y = y1;
    Args a16 = a; a16.ci = ci16; a16.slab = sb; a16.slab_shift = shift; a16.y = y1;
    int g;
    if (getenv("COOP")) {
        g_chunk_rows = 64;
        check("base u16slab 6/SM", time_us([&] { run_base<M, uint16_t, 4, 6>(a16, g); }), b16);
        g_chunk_rows = 0;
        if constexpr (M > 1) {
            check("coop u16slab G=LPR 6/SM", time_us([&] { run_coop<M, uint16_t, 6, 1>(a16); }), b16);
            check("coop u16slab G=LPR 5/SM", time_us([&] { run_coop<M, uint16_t, 5, 1>(a16); }), b16);
            check("coop u16slab G=2LPR 5/SM", time_us([&] { run_coop<M, uint16_t, 5, 2>(a16); }), b16);
            check("coop u16slab G=2LPR 4/SM", time_us([&] { run_coop<M, uint16_t, 4, 2>(a16); }), b16);
            check("coop u32 G=LPR 6/SM", time_us([&] { run_coop<M, uint32_t, 6, 1>(a32); }), b32);
        }
        return;
    }
    if (getenv("OWN")) {
        g_chunk_rows = 64;
        check("base u16slab (cold)", time_us([&] { run_base<M, uint16_t, 4, 6>(a16, g); }), b16);
        check("base u16slab (b2b, L2-warm)", time_b2b_us([&] { run_base<M, uint16_t, 4, 6>(a16, g); }), b16);
        const float t = time_us([&] { run_base<M, uint16_t, 4, 6, 1>(a16, g); });
        printf("  %-40s %9.2f us  %6.0f GB/s\n", "own-row gather (cold, no real gather)", t, b16 / t / 1e3);
        CK(cudaMemset(y1, 0, hx.size() * 8));
        g_chunk_rows = 0;
        return;
    }
    if (getenv("G4")) {
        g_chunk_rows = 64;
        check("base u16slab 6/SM chunk 64", time_us([&] { run_base<M, uint16_t, 4, 6>(a16, g); }), b16);
        check("base u32 6/SM chunk 64", time_us([&] { run_base<M, uint32_t, 4, 6>(a32, g); }), b32);
        g_chunk_rows = 0;
        constexpr int C = 32 / Lay<M>::LPR;
        std::vector<int> sp; std::vector<uint8_t> sl; std::vector<uint32_t> s32; std::vector<double> sv;
        to_g4<uint32_t>(A, A.ci, C, sp, sl, s32, sv);
        printf("  g4 C=%d padding x%.3f\n", C, (double)sv.size() / A.v.size());
        int* dsp = up(sp); uint8_t* dsl = up(sl); uint32_t* ds32 = up(s32); double* dsv = up(sv);
        Args s1 = a32; s1.ci = ds32; s1.v = dsv; s1.sptr = dsp; s1.slen = dsl;
        const double bs32 = (double)sv.size() * 12 + A.n * 1.0 + sp.size() * 4.0 + 3.0 * A.n * M * 8;
        check("g4 u32 6/SM", time_us([&] { run_g4<M, uint32_t, 6, 0>(s1); }), bs32);
        check("g4 u32 6/SM pipe", time_us([&] { run_g4<M, uint32_t, 6, 1>(s1); }), bs32);
        check("g4 u32 5/SM pipe", time_us([&] { run_g4<M, uint32_t, 5, 1>(s1); }), bs32);
        if (slab) {
            std::vector<uint16_t> s16; std::vector<double> sv2;
            to_g4<uint16_t>(A, c16, C, sp, sl, s16, sv2);
            uint16_t* ds16 = up(s16, 128);
            Args s2 = s1; s2.ci = ds16; s2.slab = sb; s2.slab_shift = shift;
            const double bs16 = (double)sv.size() * 10 + A.n * 1.0 + sp.size() * 4.0 + 3.0 * A.n * M * 8;
            check("g4 u16 6/SM", time_us([&] { run_g4<M, uint16_t, 6, 0>(s2); }), bs16);
            check("g4 u16 6/SM pipe", time_us([&] { run_g4<M, uint16_t, 6, 1>(s2); }), bs16);
            check("g4 u16 8/SM pipe", time_us([&] { run_g4<M, uint16_t, 8, 1>(s2); }), bs16);
            check("g4 u16 5/SM pipe", time_us([&] { run_g4<M, uint16_t, 5, 1>(s2); }), bs16);
            cudaFree(ds16);
        }
        cudaFree(dsp); cudaFree(dsl); cudaFree(ds32); cudaFree(dsv);
        return;
    }
    if (getenv("PF")) {
        g_chunk_rows = 64;
        check("base u16slab 6/SM chunk 64", time_us([&] { run_base<M, uint16_t, 4, 6>(a16, g); }), b16);
        g_chunk_rows = 0;
        check("pf1 u16slab UNR4 6/SM", time_us([&] { run_pf<M, uint16_t, 4, 6, 1>(a16); }), b16);
        check("pf2 u16slab UNR4 6/SM", time_us([&] { run_pf<M, uint16_t, 4, 6, 2>(a16); }), b16);
        check("pf2 u16slab UNR4 5/SM", time_us([&] { run_pf<M, uint16_t, 4, 5, 2>(a16); }), b16);
        check("pf1 u16slab UNR4 8/SM", time_us([&] { run_pf<M, uint16_t, 4, 8, 1>(a16); }), b16);
        check("pf1 u32 UNR4 6/SM", time_us([&] { run_pf<M, uint32_t, 4, 6, 1>(a32); }), b32);
        return;
    }
    if (getenv("CHUNKS")) {
        for (int cr : {32, 64, 128, 256, 512, 1024, 2048, 4096}) {
            g_chunk_rows = cr;
            char nm[64];
            snprintf(nm, 64, "base u16slab 6/SM chunk %d rows", cr);
            check(nm, time_us([&] { run_base<M, uint16_t, 4, 6>(a16, g); }), b16);
        }
        g_chunk_rows = 0;
        return;
    }
    check("base u32 (UNR4, 6/SM)", time_us([&] { run_base<M, uint32_t, 4, 6>(a32, g); }), b32);
    if (slab) check("base u16slab (UNR4, 6/SM)", time_us([&] { run_base<M, uint16_t, 4, 6>(a16, g); }), b16);
    if (slab) check("base u16slab (UNR4, 8/SM)", time_us([&] { run_base<M, uint16_t, 4, 8>(a16, g); }), b16);
    if (slab) check("base u16slab (UNR2, 8/SM)", time_us([&] { run_base<M, uint16_t, 2, 8>(a16, g); }), b16);
    if (slab) check("base u16slab (UNR8, 4/SM)", time_us([&] { run_base<M, uint16_t, 8, 4>(a16, g); }), b16);
    auto T = [&](const char* nm, float us, double byts) { if (us > 0) check(nm, us, byts); };
    {
        constexpr int C = 32 / Lay<M>::LPR;
        std::vector<int> sp; std::vector<uint8_t> sl; std::vector<uint32_t> s32; std::vector<double> sv;
        to_sell<uint32_t>(A, A.ci, C, sp, sl, s32, sv);
        const double pad = (double)sv.size() / A.v.size();
        int* dsp = up(sp); uint8_t* dsl = up(sl); uint32_t* ds32 = up(s32); double* dsv = up(sv);
        Args s1 = a32; s1.ci = ds32; s1.v = dsv; s1.sptr = dsp; s1.slen = dsl;
        printf("  sell C=%d padding x%.3f\n", C, pad);
        const double bs32 = (double)sv.size() * 12 + A.n * 1.0 + sp.size() * 4.0 + 3.0 * A.n * M * 8;
        check("sell u32 UNR4 6/SM", time_us([&] { run_sell<M, uint32_t, 4, 6>(s1); }), bs32);
        check("sell u32 UNR8 4/SM", time_us([&] { run_sell<M, uint32_t, 8, 4>(s1); }), bs32);
        if (slab) {
            std::vector<uint16_t> s16; std::vector<double> sv2;
            to_sell<uint16_t>(A, c16, C, sp, sl, s16, sv2);
            uint16_t* ds16 = up(s16, 128);
            Args s2 = s1; s2.ci = ds16; s2.slab = sb; s2.slab_shift = shift;
            const double bs16 = (double)sv.size() * 10 + A.n * 1.0 + sp.size() * 4.0 + 3.0 * A.n * M * 8;
            check("sell u16 UNR4 6/SM", time_us([&] { run_sell<M, uint16_t, 4, 6>(s2); }), bs16);
            check("sell u16 UNR8 4/SM", time_us([&] { run_sell<M, uint16_t, 8, 4>(s2); }), bs16);
            check("sell u16 UNR4 8/SM", time_us([&] { run_sell<M, uint16_t, 4, 8>(s2); }), bs16);
            cudaFree(ds16);
        }
        cudaFree(dsp); cudaFree(dsl); cudaFree(ds32); cudaFree(dsv);
    }
    if (getenv("NO_TMA")) goto done;
    T("tma u32 NCW8 S6 UNR8 2/SM", try_tma<M, uint32_t, 8, 6, EPR, 8>(a32, 0, 2), b32);
    T("tma u32 NCW8 S6 UNR8 max/SM", try_tma<M, uint32_t, 8, 6, EPR, 8>(a32, 0, 0), b32);
    T("tma u32 NCW8 S4 UNR8 max/SM", try_tma<M, uint32_t, 8, 4, EPR, 8>(a32, 0, 0), b32);
    T("tma u32 NCW4 S4 UNR8 max/SM", try_tma<M, uint32_t, 4, 4, EPR, 8>(a32, 0, 0), b32);
    if (slab) {
        T("tma u16 NCW8 S6 UNR8 max/SM", try_tma<M, uint16_t, 8, 6, EPR, 8>(a16, 0, 0), b16);
        T("tma u16 NCW8 S4 UNR8 max/SM", try_tma<M, uint16_t, 8, 4, EPR, 8>(a16, 0, 0), b16);
        T("tma u16 NCW16 S4 UNR8 max/SM", try_tma<M, uint16_t, 16, 4, EPR, 8>(a16, 0, 0), b16);
        T("tma u16 NCW8 S6 UNR4 max/SM", try_tma<M, uint16_t, 8, 6, EPR, 4>(a16, 0, 0), b16);
        T("tma u16 NCW4 S8 UNR8 max/SM", try_tma<M, uint16_t, 4, 8, EPR, 8>(a16, 0, 0), b16);
        T("tma u16 NCW4 S4 UNR8 max/SM", try_tma<M, uint16_t, 4, 4, EPR, 8>(a16, 0, 0), b16);
        T("tma u16 NCW8 S6 UNR8 tpc1", try_tma<M, uint16_t, 8, 6, EPR, 8>(a16, 1, 0), b16);
        T("tma u16 NCW8 S6 UNR8 tpc32", try_tma<M, uint16_t, 8, 6, EPR, 8>(a16, 32, 0), b16);
    }
done:
    cudaFree(x); cudaFree(b); cudaFree(y0); cudaFree(y1); cudaFree(rp); cudaFree(ci32); cudaFree(v);
    if (ci16) cudaFree(ci16);
    if (sb) cudaFree(sb);
}


__global__ void k_empty(int* p) { if (p && threadIdx.x == 1023) p[0] = 1; }

static void graph_gap() {
    cudaStream_t st;
    cudaStreamCreate(&st);
    for (int grid : {1, 148, 888}) {
        cudaGraph_t g;
        cudaGraphExec_t ge;
        CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal));
        for (int i = 0; i < 200; ++i) k_empty<<<grid, 256, 0, st>>>(nullptr);
        CK(cudaStreamEndCapture(st, &g));
        CK(cudaGraphInstantiate(&ge, g, 0));
        CK(cudaGraphLaunch(ge, st));
        CK(cudaStreamSynchronize(st));
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0, st);
        for (int r = 0; r < 10; ++r) CK(cudaGraphLaunch(ge, st));
        cudaEventRecord(e1, st);
        CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("graph of 200 empty kernels, grid %d: %.3f us per kernel\n", grid, ms * 1e3 / 2000);
    }
}


__global__ void k_loopctl(cudaGraphConditionalHandle h, int* cnt, int iters) {
    int c = ++cnt[0];
    cudaGraphSetConditional(h, c < iters ? 1u : 0u);
}

static void while_gap() {
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    int* cnt;
    CK(cudaMalloc(&cnt, 4));
    for (int body : {1, 16}) {
        const int iters = 200 / body;
        cudaGraph_t g;
        CK(cudaGraphCreate(&g, 0));
        cudaGraphConditionalHandle h;
        CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t wnode;
        CK(cudaGraphAddNode(&wnode, g, nullptr, 0, &cp));
        cudaGraph_t bodyg = cp.conditional.phGraph_out[0];
        CK(cudaStreamBeginCaptureToGraph(st, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
        for (int i = 0; i < body - 1; ++i) k_empty<<<888, 256, 0, st>>>(nullptr);
        k_loopctl<<<1, 1, 0, st>>>(h, cnt, iters);
        cudaGraph_t tmp;
        CK(cudaStreamEndCapture(st, &tmp));
        cudaGraphExec_t ge;
        CK(cudaGraphInstantiate(&ge, g, 0));
        CK(cudaMemset(cnt, 0, 4));
        CK(cudaGraphLaunch(ge, st));
        CK(cudaStreamSynchronize(st));
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        const int R = 5;
        float tot = 0;
        for (int r = 0; r < R; ++r) {
            CK(cudaMemset(cnt, 0, 4));
            CK(cudaStreamSynchronize(st));
            cudaEventRecord(e0, st);
            CK(cudaGraphLaunch(ge, st));
            cudaEventRecord(e1, st);
            CK(cudaEventSynchronize(e1));
            float ms; cudaEventElapsedTime(&ms, e0, e1); tot += ms;
        }
        printf("WHILE loop, body of %d kernels (grid 888 + 1-thread control), %d iterations: %.3f us per iteration, %.3f us per kernel\n",
               body, iters, tot / R * 1e3 / iters, tot / R * 1e3 / (iters * body));
    }
}

int main(int argc, char** argv) {
    CK(cudaMalloc(&g_flush, 256u << 20));
    const char* which = argc > 1 ? argv[1] : "all";
    auto want = [&](const char* k) { return !strcmp(which, "all") || strstr(which, k); };
    if (!strcmp(which, "gap")) { graph_gap(); while_gap(); return 0; }
    if (want("c2")) { Csr A = poisson7(64); bench_matrix<8, 8>(A); }
    if (want("c3")) { Csr A = poisson7(128); bench_matrix<16, 8>(A); bench_matrix<8, 8>(A); }
    if (want("c4")) { Csr A = stencil27(128); bench_matrix<8, 32>(A); }
    if (want("c5")) { Csr A = band_random(1 << 22, 4096, 15.0); bench_matrix<8, 24>(A); bench_matrix<1, 24>(A); }
    return 0;
}
