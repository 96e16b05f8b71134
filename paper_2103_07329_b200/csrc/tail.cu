// tail.cu -- instantiation and cluster launch of the V-cycle tail kernel.
#include "launch.cuh"
#include "tail.cuh"

namespace mrs {

template <int M>
static cudaError_t tail_launch_m(const TailStep* steps, int nsteps, const int* guard, int csize,
                                 cudaStream_t s) {
    auto kern = tail_kernel<M>;
    static int attr_done = 0;
    if (!attr_done) {
        cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        attr_done = 1;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(csize);
    cfg.blockDim = dim3(kThreads);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = csize;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, steps, nsteps, guard);
}

// Largest supported cluster (16 non-portable, else 8) for this m.
int tail_cluster_size(int64_t m) {
    static int cached[65] = {0};
    if (m < 1 || m > 64) return 0;
    if (cached[m]) return cached[m];
    const void* fn = nullptr;
    switch (m) {
    case 1: fn = (const void*)tail_kernel<1>; break;
    case 2: fn = (const void*)tail_kernel<2>; break;
    case 4: fn = (const void*)tail_kernel<4>; break;
    case 8: fn = (const void*)tail_kernel<8>; break;
    case 16: fn = (const void*)tail_kernel<16>; break;
    case 32: fn = (const void*)tail_kernel<32>; break;
    case 64: fn = (const void*)tail_kernel<64>; break;
    default: return 0;
    }
    int best = 0;
    cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs : {16, 8, 4}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cs);
        cfg.blockDim = dim3(kThreads);
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = cs;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int nclusters = 0;
        if (cudaOccupancyMaxActiveClusters(&nclusters, fn, &cfg) == cudaSuccess && nclusters > 0) {
            best = cs;
            break;
        }
    }
    cudaGetLastError();
    cached[m] = best;
    return best;
}

cudaError_t launch_tail(const TailStep* steps, int nsteps, int64_t m, const int* guard, int csize,
                        cudaStream_t s) {
    switch (m) {
    case 1: return tail_launch_m<1>(steps, nsteps, guard, csize, s);
    case 2: return tail_launch_m<2>(steps, nsteps, guard, csize, s);
    case 4: return tail_launch_m<4>(steps, nsteps, guard, csize, s);
    case 8: return tail_launch_m<8>(steps, nsteps, guard, csize, s);
    case 16: return tail_launch_m<16>(steps, nsteps, guard, csize, s);
    case 32: return tail_launch_m<32>(steps, nsteps, guard, csize, s);
    case 64: return tail_launch_m<64>(steps, nsteps, guard, csize, s);
    }
    return cudaErrorInvalidValue;
}

}  // namespace mrs
