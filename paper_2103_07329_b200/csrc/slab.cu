// slab.cu -- index compression of an uploaded operator ON THE DEVICE (setup
// phase): 32-bit columns -> slab-relative 16-bit ones, the same rule and the
// same result as the host routine core.slab_compress (rows in slabs of 2^shift
// rows, every entry stores column - base[slab], base = the slab's smallest
// column, the largest shift in [6, 24] whose slabs all span < 65536 columns).
// The host version costs ~4 s per 56 M entries in numpy (C4 at 128^3: 40 % of
// prepare); here the column stream is read twice at HBM speed.
#include <algorithm>
#include <climits>
#include <vector>

#include "dispatch.h"

namespace mrs {

namespace {

// one warp per group of 64 consecutive rows: min / max column of its entries
__global__ void slab6_minmax_kernel(const int32_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                                    int64_t nrows, int64_t ngroups, int32_t* __restrict__ gmin,
                                    int32_t* __restrict__ gmax) {
    const int lane = threadIdx.x % 32;
    for (int64_t g = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; g < ngroups;
         g += (int64_t)gridDim.x * (blockDim.x / 32)) {
        const int64_t r0 = g * 64, r1 = min(nrows, r0 + 64);
        const int e0 = rp[r0], e1 = rp[r1];
        int mn = INT_MAX, mx = -1;
        for (int e = e0 + lane; e < e1; e += 32) {
            const int c = (int)ci[e];
            mn = min(mn, c); mx = max(mx, c);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mn = min(mn, __shfl_xor_sync(~0u, mn, o));
            mx = max(mx, __shfl_xor_sync(~0u, mx, o));
        }
        if (lane == 0) { gmin[g] = mn; gmax[g] = mx; }
    }
}

__global__ void slab_convert_kernel(const int32_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                                    int64_t nrows, int64_t ngroups, const int32_t* __restrict__ base,
                                    int shift, uint16_t* __restrict__ out) {
    const int lane = threadIdx.x % 32;
    for (int64_t g = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; g < ngroups;
         g += (int64_t)gridDim.x * (blockDim.x / 32)) {
        const int64_t r0 = g * 64, r1 = min(nrows, r0 + 64);
        const int e0 = rp[r0], e1 = rp[r1];
        const int b = base[r0 >> shift];
        for (int e = e0 + lane; e < e1; e += 32) out[e] = (uint16_t)((int)ci[e] - b);
    }
}

}  // namespace

// Returns 1 and fills (ci16, base, shift, nslabs) -- device arrays the caller
// owns -- when the columns fit slab-relative 16 bits; 0 when they do not; -1 on
// a CUDA error.  rp_dev / ci32_dev: the uploaded row pointers and columns.
int slab_compress_device(const int32_t* rp_dev, const uint32_t* ci32_dev, int64_t nrows, int64_t nnz,
                         int64_t ncols, uint16_t** ci16, int32_t** base, int* shift,
                         int64_t* nslabs) {
    constexpr int kMinShift = 6, kMaxShift = 24;
    if (nrows <= 0 || nnz <= 0 || ncols >= (1ll << 31)) return 0;
    const int64_t ng = (nrows + 63) / 64;
    int32_t *gmin = nullptr, *gmax = nullptr;
    if (cudaMalloc(&gmin, ng * 4) != cudaSuccess || cudaMalloc(&gmax, ng * 4) != cudaSuccess) {
        if (gmin) cudaFree(gmin);
        cudaGetLastError();
        return -1;
    }
    const int grid = (int)std::min<int64_t>((ng + 7) / 8, (int64_t)num_sms() * 8);
    slab6_minmax_kernel<<<grid, 256>>>(rp_dev, ci32_dev, nrows, ng, gmin, gmax);
    std::vector<int32_t> mn(ng), mx(ng);
    const bool ok = cudaMemcpy(mn.data(), gmin, ng * 4, cudaMemcpyDeviceToHost) == cudaSuccess &&
                    cudaMemcpy(mx.data(), gmax, ng * 4, cudaMemcpyDeviceToHost) == cudaSuccess;
    cudaFree(gmin); cudaFree(gmax);
    if (!ok) { cudaGetLastError(); return -1; }
    // slab extremes for shift = 6, 7, ..., 24 by pairwise merging; keep the largest fitting
    std::vector<int32_t> best_base;
    int best_shift = -1;
    std::vector<int32_t> cmn = mn, cmx = mx;
    for (int s = kMinShift; s <= kMaxShift; ++s) {
        if (s > kMinShift) {
            const size_t h = (cmn.size() + 1) / 2;
            std::vector<int32_t> nmn(h), nmx(h);
            for (size_t i = 0; i < h; ++i) {
                const size_t a = 2 * i, b = 2 * i + 1;
                nmn[i] = b < cmn.size() ? std::min(cmn[a], cmn[b]) : cmn[a];
                nmx[i] = b < cmx.size() ? std::max(cmx[a], cmx[b]) : cmx[a];
            }
            cmn.swap(nmn); cmx.swap(nmx);
        }
        bool fits = true;
        for (size_t i = 0; i < cmn.size() && fits; ++i)
            if (cmx[i] >= 0 && (int64_t)cmx[i] - cmn[i] >= 65536) fits = false;
        if (!fits) break;                // spans only grow with the slab size
        best_shift = s;
        best_base.resize(cmn.size());
        for (size_t i = 0; i < cmn.size(); ++i) best_base[i] = cmx[i] < 0 ? 0 : cmn[i];
    }
    if (best_shift < 0) return 0;
    // (the number of slabs of the chosen shift: ceil(nrows / 2^shift))
    const int64_t ns = ((nrows - 1) >> best_shift) + 1;
    if ((int64_t)best_base.size() < ns) return -1;
    uint16_t* o16 = nullptr;
    int32_t* bdev = nullptr;
    if (cudaMalloc(&o16, nnz * 2) != cudaSuccess || cudaMalloc(&bdev, ns * 4) != cudaSuccess) {
        if (o16) cudaFree(o16);
        cudaGetLastError();
        return -1;
    }
    if (cudaMemcpy(bdev, best_base.data(), ns * 4, cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaFree(o16); cudaFree(bdev);
        return -1;
    }
    slab_convert_kernel<<<grid, 256>>>(rp_dev, ci32_dev, nrows, ng, bdev, best_shift, o16);
    if (cudaDeviceSynchronize() != cudaSuccess) {
        cudaFree(o16); cudaFree(bdev);
        cudaGetLastError();
        return -1;
    }
    *ci16 = o16; *base = bdev; *shift = best_shift; *nslabs = ns;
    return 1;
}

}  // namespace mrs
