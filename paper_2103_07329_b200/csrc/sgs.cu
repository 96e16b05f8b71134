// sgs.cu -- instantiation and cluster launch of the Gauss-Seidel half-sweep
// kernel (sgs.cuh).
#include "launch.cuh"
#include "sgs.cuh"

namespace mrs {

template <int CPL, typename Tv, typename Ti>
static int sgs_cluster_size() {
    static int best = -1;
    if (best >= 0) return best;
    const void* fn = (const void*)sgs_kernel<CPL, Tv, Ti>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    best = 0;
    for (int cs : {16, 8, 4, 2, 1}) {
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
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) == cudaSuccess && n > 0) {
            best = cs;
            break;
        }
    }
    cudaGetLastError();
    return best;
}

template <int CPL, typename Tv, typename Ti>
static cudaError_t sgs_launch_t(const SgsArgs& a, cudaStream_t s) {
    // one CTA when a schedule level averages at most one CTA pass of rows
    const int64_t cta_rows = kSgsCta / (a.m / CPL);
    if ((int64_t)a.nrows <= cta_rows * a.nlev) {
        sgs_cta_kernel<CPL, Tv, Ti><<<1, kSgsCta, 0, s>>>(a);
        return cudaGetLastError();
    }
    const int cs = sgs_cluster_size<CPL, Tv, Ti>();
    if (cs < 1) return cudaErrorLaunchOutOfResources;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(kThreads);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, sgs_kernel<CPL, Tv, Ti>, a);
}

template <int CPL>
static cudaError_t sgs_launch_c(const SgsArgs& a, int vb, int ib, cudaStream_t s) {
    if (vb == 8) {
        if (ib == 2) return sgs_launch_t<CPL, double, uint16_t>(a, s);
        if (ib == 4) return sgs_launch_t<CPL, double, uint32_t>(a, s);
    } else if (vb == 4) {
        if (ib == 2) return sgs_launch_t<CPL, float, uint16_t>(a, s);
        if (ib == 4) return sgs_launch_t<CPL, float, uint32_t>(a, s);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_sgs(const SgsArgs& a, int vb, int ib, cudaStream_t s) {
    if (a.m < 1 || a.m > kThreads) return cudaErrorInvalidValue;
    if (a.nlev == 0) return cudaSuccess;
    return (a.m % 2 == 0) ? sgs_launch_c<2>(a, vb, ib, s) : sgs_launch_c<1>(a, vb, ib, s);
}

}  // namespace mrs
