// spgemm.cu -- Galerkin product A_c = (R A) P of the AMG setup on the GPU
// (reference src/amg.py:185-196 = scipy csr_matmat).
//
// One output row per warp (rows whose product count is <= 1024: hash table of
// 2048 slots in shared memory) or per CTA (longer rows: table in global scratch).
// The left row's entries are walked SEQUENTIALLY (jj), the right row's entries
// of one jj in parallel (kk, distinct columns): each output column receives its
// products in jj order with separately rounded multiply and add, i.e. the sums
// of scipy's SMMP kernel bit for bit.  Exact zeros are dropped.  order 0 emits a
// row in scipy's order (reverse first touch: the intermediate R A, whose row
// order is the summation order of the second product), order 1 sorted by column.
// Two passes: count, exclusive scan (cub), fill.
#include "spgemm.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cub/device/device_scan.cuh>
#include <thread>

namespace mrs {

namespace {

constexpr int kT1Cap = 2048;      // hash slots per warp (tier 1)
constexpr int kT1Max = 1024;      // most products (hence distinct columns) of a tier-1 row
constexpr int kT1Warps = 4;
constexpr int kT2Threads = 256;

struct DCsr {
    int64_t nrows = 0, ncols = 0, nnz = 0;
    int64_t* rp = nullptr;
    int32_t* ci = nullptr;
    double* v = nullptr;
    void release() {
        if (rp) cudaFree(rp);
        if (ci) cudaFree(ci);
        if (v) cudaFree(v);
        rp = nullptr; ci = nullptr; v = nullptr;
    }
};

struct Buf {                       // owning device allocation
    void* p = nullptr;
    ~Buf() { if (p) cudaFree(p); }
    bool alloc(size_t bytes) { return cudaMalloc(&p, bytes ? bytes : 16) == cudaSuccess; }
    template <typename T> T* as() { return reinterpret_cast<T*>(p); }
};

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }

__global__ void narrow_kernel(const int64_t* __restrict__ in, int32_t* __restrict__ out, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int32_t)in[i];
}
__global__ void widen_kernel(const int32_t* __restrict__ in, int64_t* __restrict__ out, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = in[i];
}

// products of row i: sum over its entries of the right operand's row lengths
__global__ void ub_kernel(int64_t n, const int64_t* __restrict__ arp, const int32_t* __restrict__ aci,
                          const int64_t* __restrict__ brp, int64_t* __restrict__ ub) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t s = 0;
        for (int64_t jj = arp[i]; jj < arp[i + 1]; ++jj) {
            const int j = aci[jj];
            s += brp[j + 1] - brp[j];
        }
        ub[i] = s;
    }
}

struct PArgs {
    const int64_t* arp; const int32_t* aci; const double* av;
    const int64_t* brp; const int32_t* bci; const double* bv;
    const int32_t* rows; int nlist;       // rows of this tier
    int fill, order;                      // fill: 0 = count pass
    int64_t* cnt;                         // per row (count pass)
    const int64_t* crp; int32_t* cci; double* cv;
    // tier 2 scratch, per CTA: keys | seq | skey | scol (int32 x cap2) , vals | sval (double x cap2)
    int32_t* s_i32; double* s_f64; const int64_t* ub; int cap2;
};

__device__ __forceinline__ uint32_t hash_slot(int k, int log2cap) {
    return ((uint32_t)k * 2654435761u) >> (32 - log2cap);
}

// insert-or-find column k; returns its slot.  Concurrent callers hold DISTINCT k.
__device__ __forceinline__ int table_slot(int32_t* keys, int32_t* seq, int k, int sq, int cap,
                                          int log2cap) {
    uint32_t h = hash_slot(k, log2cap);
    while (true) {
        const int old = atomicCAS(&keys[h], -1, k);
        if (old == -1) { seq[h] = sq; return (int)h; }
        if (old == k) return (int)h;
        h = (h + 1) & (uint32_t)(cap - 1);
    }
}

// ---- tier 1: one warp per row, table and sort buffer in shared memory
__global__ void __launch_bounds__(kT1Warps * 32) spgemm_warp_kernel(PArgs a) {
    extern __shared__ __align__(16) unsigned char sm[];
    constexpr int CAP = kT1Cap, CB = kT1Max, L2 = 11;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    unsigned char* base = sm + (size_t)warp * (CAP * 16 + CB * 16);
    double* vals = reinterpret_cast<double*>(base);
    int32_t* keys = reinterpret_cast<int32_t*>(base + CAP * 8);
    int32_t* seq = keys + CAP;
    double* oval = reinterpret_cast<double*>(base + CAP * 16);
    int32_t* okey = reinterpret_cast<int32_t*>(base + CAP * 16 + CB * 8);
    int32_t* ocol = okey + CB;
    for (int it = blockIdx.x * kT1Warps + warp; it < a.nlist; it += gridDim.x * kT1Warps) {
        const int i = a.rows[it];
        for (int s = lane; s < CAP; s += 32) { keys[s] = -1; vals[s] = 0.0; }
        __syncwarp();
        int sq0 = 0;
        for (int64_t jj = a.arp[i]; jj < a.arp[i + 1]; ++jj) {
            const int j = a.aci[jj];
            const double av = a.av[jj];
            const int64_t b0 = a.brp[j];
            const int lb = (int)(a.brp[j + 1] - b0);
            for (int kk0 = 0; kk0 < lb; kk0 += 32) {
                const int kk = kk0 + lane;
                if (kk < lb) {
                    const int k = a.bci[b0 + kk];
                    const double p = dmul(av, a.bv[b0 + kk]);
                    const int h = table_slot(keys, seq, k, sq0 + kk, CAP, L2);
                    vals[h] = dadd(vals[h], p);
                }
                __syncwarp();
            }
            sq0 += lb;
        }
        // count / compact the nonzero sums
        int run = 0;
        for (int s0 = 0; s0 < CAP; s0 += 32) {
            const int s = s0 + lane;
            const bool on = keys[s] >= 0 && vals[s] != 0.0;
            const unsigned m = __ballot_sync(~0u, on);
            if (a.fill && on) {
                const int pos = run + __popc(m & ((1u << lane) - 1));
                okey[pos] = a.order ? keys[s] : INT_MAX - 1 - seq[s];
                ocol[pos] = keys[s];
                oval[pos] = vals[s];
            }
            run += __popc(m);
        }
        if (!a.fill) {
            if (lane == 0) a.cnt[i] = run;
            __syncwarp();
            continue;
        }
        int n2 = 1;
        while (n2 < run) n2 <<= 1;
        for (int t = run + lane; t < n2; t += 32) okey[t] = INT_MAX;
        __syncwarp();
        for (int k = 2; k <= n2; k <<= 1)
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int t = lane; t < n2; t += 32) {
                    const int x = t ^ j;
                    if (x > t) {
                        const bool up = (t & k) == 0;
                        const int kt = okey[t], kx = okey[x];
                        if ((kt > kx) == up) {
                            okey[t] = kx; okey[x] = kt;
                            const int ct = ocol[t]; ocol[t] = ocol[x]; ocol[x] = ct;
                            const double vt = oval[t]; oval[t] = oval[x]; oval[x] = vt;
                        }
                    }
                }
                __syncwarp();
            }
        const int64_t o = a.crp[i];
        for (int t = lane; t < run; t += 32) { a.cci[o + t] = ocol[t]; a.cv[o + t] = oval[t]; }
        __syncwarp();
    }
}

// ---- tier 2: one CTA per row, table and sort buffer in global scratch
__global__ void __launch_bounds__(kT2Threads) spgemm_cta_kernel(PArgs a) {
    __shared__ int s_cnt;
    const int tid = threadIdx.x;
    int32_t* keys = a.s_i32 + (size_t)blockIdx.x * 4 * a.cap2;
    int32_t* seq = keys + a.cap2;
    int32_t* skey = seq + a.cap2;
    int32_t* scol = skey + a.cap2;
    double* vals = a.s_f64 + (size_t)blockIdx.x * 2 * a.cap2;
    double* sval = vals + a.cap2;
    for (int it = blockIdx.x; it < a.nlist; it += gridDim.x) {
        const int i = a.rows[it];
        int cap = 4096, l2 = 12;
        while (cap < 2 * a.ub[i]) { cap <<= 1; ++l2; }      // <= cap2 (host sized it)
        for (int s = tid; s < cap; s += kT2Threads) { keys[s] = -1; vals[s] = 0.0; }
        if (tid == 0) s_cnt = 0;
        __syncthreads();
        int sq0 = 0;
        for (int64_t jj = a.arp[i]; jj < a.arp[i + 1]; ++jj) {
            const int j = a.aci[jj];
            const double av = a.av[jj];
            const int64_t b0 = a.brp[j];
            const int lb = (int)(a.brp[j + 1] - b0);
            for (int kk = tid; kk < lb; kk += kT2Threads) {
                const int k = a.bci[b0 + kk];
                const double p = dmul(av, a.bv[b0 + kk]);
                const int h = table_slot(keys, seq, k, sq0 + kk, cap, l2);
                vals[h] = dadd(vals[h], p);
            }
            __syncthreads();
            sq0 += lb;
        }
        for (int s = tid; s < cap; s += kT2Threads) {
            if (keys[s] >= 0 && vals[s] != 0.0) {
                const int pos = atomicAdd(&s_cnt, 1);          // any order: sorted below
                if (a.fill) {
                    skey[pos] = a.order ? keys[s] : INT_MAX - 1 - seq[s];
                    scol[pos] = keys[s];
                    sval[pos] = vals[s];
                }
            }
        }
        __syncthreads();
        const int run = s_cnt;
        if (!a.fill) {
            if (tid == 0) a.cnt[i] = run;
            __syncthreads();
            continue;
        }
        int n2 = 1;
        while (n2 < run) n2 <<= 1;
        for (int t = run + tid; t < n2; t += kT2Threads) skey[t] = INT_MAX;
        __syncthreads();
        for (int k = 2; k <= n2; k <<= 1)
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int t = tid; t < n2; t += kT2Threads) {
                    const int x = t ^ j;
                    if (x > t) {
                        const bool up = (t & k) == 0;
                        const int kt = skey[t], kx = skey[x];
                        if ((kt > kx) == up) {
                            skey[t] = kx; skey[x] = kt;
                            const int ct = scol[t]; scol[t] = scol[x]; scol[x] = ct;
                            const double vt = sval[t]; sval[t] = sval[x]; sval[x] = vt;
                        }
                    }
                }
                __syncthreads();
            }
        const int64_t o = a.crp[i];
        for (int t = tid; t < run; t += kT2Threads) { a.cci[o + t] = scol[t]; a.cv[o + t] = sval[t]; }
        __syncthreads();
    }
}

// fn(lo, hi) over contiguous ranges of [0, n) on host threads
template <class Fn> void host_parallel(int64_t n, Fn fn) {
    const int parts = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    if (parts <= 1 || n < (1 << 16)) { fn((int64_t)0, n); return; }
    std::vector<std::thread> th;
    for (int p = 0; p < parts; ++p) {
        const int64_t lo = n * p / parts, hi = n * (p + 1) / parts;
        th.emplace_back([=, &fn] { fn(lo, hi); });
    }
    for (auto& t : th) t.join();
}

int sm_count() {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms > 0 ? sms : 148;
}

bool upload(const HostCsrView& H, DCsr& D) {
    D.nrows = H.nrows; D.ncols = H.ncols; D.nnz = H.rp[H.nrows];
    if (H.ncols >= INT32_MAX || H.nrows >= INT32_MAX) return false;
    if (cudaMalloc(&D.rp, (H.nrows + 1) * 8) != cudaSuccess) return false;
    if (cudaMalloc(&D.ci, std::max<int64_t>(D.nnz, 1) * 4) != cudaSuccess) return false;
    if (cudaMalloc(&D.v, std::max<int64_t>(D.nnz, 1) * 8) != cudaSuccess) return false;
    if (cudaMemcpy(D.rp, H.rp, (H.nrows + 1) * 8, cudaMemcpyHostToDevice) != cudaSuccess) return false;
    if (D.nnz) {
        // columns narrowed to 32 bits on the host threads: half the PCIe bytes
        std::vector<int32_t> c32((size_t)D.nnz);
        const int64_t* src = H.ci;
        host_parallel(D.nnz, [&](int64_t lo, int64_t hi) {
            for (int64_t k = lo; k < hi; ++k) c32[k] = (int32_t)src[k];
        });
        if (cudaMemcpy(D.ci, c32.data(), D.nnz * 4, cudaMemcpyHostToDevice) != cudaSuccess) return false;
        if (cudaMemcpy(D.v, H.v, D.nnz * 8, cudaMemcpyHostToDevice) != cudaSuccess) return false;
    }
    return cudaDeviceSynchronize() == cudaSuccess;
}

// C = A * B on the device (see the file header for `order`).
bool product(const DCsr& A, const DCsr& B, int order, DCsr& Cm) {
    const int64_t n = A.nrows;
    Cm.nrows = n; Cm.ncols = B.ncols;
    Buf ubd, cntd, l1d, l2d, tmpd, s32, s64;
    if (!ubd.alloc((n + 1) * 8) || !cntd.alloc((n + 1) * 8)) return false;
    ub_kernel<<<1024, 256>>>(n, A.rp, A.ci, B.rp, ubd.as<int64_t>());
    std::vector<int64_t> ub(n);
    if (cudaMemcpy(ub.data(), ubd.p, n * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return false;
    std::vector<int32_t> l1, l2;
    int64_t ubmax = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (ub[i] <= kT1Max) l1.push_back((int32_t)i);
        else { l2.push_back((int32_t)i); ubmax = std::max(ubmax, ub[i]); }
    }
    if (ubmax >= (1ll << 28)) return false;                 // table of 2^29 slots: not here
    int cap2 = 4096;
    while (cap2 < 2 * ubmax) cap2 <<= 1;
    const int ctas2 = (int)std::min<int64_t>((int64_t)l2.size(), 2 * sm_count());
    if (!l1d.alloc(l1.size() * 4) || !l2d.alloc(l2.size() * 4)) return false;
    if (!l1.empty()) cudaMemcpy(l1d.p, l1.data(), l1.size() * 4, cudaMemcpyHostToDevice);
    if (!l2.empty()) {
        cudaMemcpy(l2d.p, l2.data(), l2.size() * 4, cudaMemcpyHostToDevice);
        if (!s32.alloc((size_t)ctas2 * 4 * cap2 * 4) || !s64.alloc((size_t)ctas2 * 2 * cap2 * 8))
            return false;
    }
    if (cudaMemset(cntd.p, 0, (n + 1) * 8) != cudaSuccess) return false;
    if (cudaMalloc(&Cm.rp, (n + 1) * 8) != cudaSuccess) return false;
    const size_t smem1 = (size_t)kT1Warps * (kT1Cap * 16 + kT1Max * 16);
    if (cudaFuncSetAttribute(spgemm_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem1) != cudaSuccess)
        return false;
    PArgs a;
    a.arp = A.rp; a.aci = A.ci; a.av = A.v; a.brp = B.rp; a.bci = B.ci; a.bv = B.v;
    a.order = order; a.cnt = cntd.as<int64_t>();
    a.crp = Cm.rp; a.cci = nullptr; a.cv = nullptr;
    a.s_i32 = s32.as<int32_t>(); a.s_f64 = s64.as<double>(); a.ub = ubd.as<int64_t>(); a.cap2 = cap2;
    auto pass = [&](int fill) {
        a.fill = fill;
        if (!l1.empty()) {
            a.rows = l1d.as<int32_t>(); a.nlist = (int)l1.size();
            const int g = (int)std::min<int64_t>(((int64_t)l1.size() + kT1Warps - 1) / kT1Warps,
                                                 (int64_t)sm_count());
            spgemm_warp_kernel<<<g, kT1Warps * 32, smem1>>>(a);
        }
        if (!l2.empty()) {
            a.rows = l2d.as<int32_t>(); a.nlist = (int)l2.size();
            spgemm_cta_kernel<<<ctas2, kT2Threads>>>(a);
        }
        return cudaDeviceSynchronize() == cudaSuccess;
    };
    if (!pass(0)) return false;
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, cntd.as<int64_t>(), Cm.rp, n + 1);
    if (!tmpd.alloc(tb)) return false;
    if (cub::DeviceScan::ExclusiveSum(tmpd.p, tb, cntd.as<int64_t>(), Cm.rp, n + 1) != cudaSuccess)
        return false;
    if (cudaMemcpy(&Cm.nnz, Cm.rp + n, 8, cudaMemcpyDeviceToHost) != cudaSuccess) return false;
    if (cudaMalloc(&Cm.ci, std::max<int64_t>(Cm.nnz, 1) * 4) != cudaSuccess) return false;
    if (cudaMalloc(&Cm.v, std::max<int64_t>(Cm.nnz, 1) * 8) != cudaSuccess) return false;
    a.cci = Cm.ci; a.cv = Cm.v;
    return pass(1);
}

std::atomic<int64_t> g_count{0};
int64_t g_enabled = -1;

}  // namespace

void set_setup_gpu(int64_t v) { g_enabled = v ? 1 : 0; }
int64_t setup_gpu() {
    if (g_enabled < 0) {
        const char* e = getenv("MRS_SETUP_GPU");
        g_enabled = (e && e[0] == '0') ? 0 : 1;
    }
    return g_enabled;
}
int64_t galerkin_gpu_count() { return g_count.load(); }

bool galerkin_gpu(const HostCsrView& R, const HostCsrView& A, const HostCsrView& P,
                  std::vector<int64_t>& rp, std::vector<int64_t>& ci, std::vector<double>& v) {
    if (!setup_gpu()) return false;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
        cudaGetLastError();
        return false;
    }
    DCsr dR, dA, dP, dRA, dC;
    const bool timing = getenv("MRS_SETUP_TIMING") != nullptr;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto secs = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
    const auto t0 = now();
    bool ok = upload(R, dR) && upload(A, dA);
    const auto t1 = now();
    ok = ok && product(dR, dA, 0, dRA);
    const auto t2 = now();
    dR.release(); dA.release();
    ok = ok && upload(P, dP) && product(dRA, dP, 1, dC);
    const auto t3 = now();
    const int64_t nnz_ra = dRA.nnz;
    dRA.release(); dP.release();
    if (ok) {
        const int64_t n = dC.nrows, nnz = dC.nnz;
        rp.resize(n + 1); ci.resize(nnz); v.resize(nnz);
        std::vector<int32_t> c32((size_t)nnz);
        ok = cudaMemcpy(rp.data(), dC.rp, (n + 1) * 8, cudaMemcpyDeviceToHost) == cudaSuccess &&
             (nnz == 0 ||
              (cudaMemcpy(c32.data(), dC.ci, nnz * 4, cudaMemcpyDeviceToHost) == cudaSuccess &&
               cudaMemcpy(v.data(), dC.v, nnz * 8, cudaMemcpyDeviceToHost) == cudaSuccess));
        if (ok)
            host_parallel(nnz, [&](int64_t lo, int64_t hi) {
                for (int64_t k = lo; k < hi; ++k) ci[k] = c32[k];
            });
    }
    dC.release();
    if (!ok) { cudaGetLastError(); return false; }
    if (timing && A.nrows > 100000)
        fprintf(stderr, "[galerkin_gpu] n %lld nnz(A) %lld nnz(RA) %lld nnz(Ac) %lld: upload %.2fs  R*A %.2fs  "
                "(RA)*P %.2fs  download %.2fs\n", (long long)A.nrows, (long long)A.rp[A.nrows],
                (long long)nnz_ra, (long long)rp.back(), secs(t0, t1), secs(t1, t2), secs(t2, t3),
                secs(t3, now()));
    g_count.fetch_add(1);
    return true;
}

}  // namespace mrs
