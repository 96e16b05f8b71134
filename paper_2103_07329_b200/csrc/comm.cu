// comm.cu -- NCCL communicator C ABI, halo exchange, split reductions.
#include <cstring>

#include "comm.h"
#include "dispatch.h"

namespace mrs {

__global__ void __launch_bounds__(kThreads) pack_kernel(const double* __restrict__ x,
                                                        const int32_t* __restrict__ idx, int n,
                                                        int m, double* __restrict__ out,
                                                        const int* guard) {
    if (guard && *guard) return;
    const int64_t total = (int64_t)n * m;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / m, c = e % m;
        out[e] = x[(int64_t)__ldg(idx + i) * m + c];
    }
}

cudaError_t halo_exchange(const Halo& h, double* x, int64_t m, const mrs_comm* c, const int* guard,
                          cudaStream_t s) {
    if (!h.active()) return cudaSuccess;
    if (h.nsend) {
        const int64_t total = (int64_t)h.nsend * m;
        int g = (int)((total + kThreads - 1) / kThreads);
        if (g > max_grid()) g = max_grid();
        pack_kernel<<<g, kThreads, 0, s>>>(x, h.send_idx, h.nsend, (int)m, h.sendbuf, guard);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    if (ncclGroupStart() != ncclSuccess) return cudaErrorUnknown;
    for (int p = 0; p < c->nranks; ++p) {
        if (h.scount[p])
            if (ncclSend(h.sendbuf + (int64_t)h.sdisp[p] * m, (size_t)h.scount[p] * m, ncclDouble, p,
                         c->comm, s) != ncclSuccess) { ncclGroupEnd(); return cudaErrorUnknown; }
        if (h.rcount[p])
            if (ncclRecv(x + (h.recv_row0 + h.rdisp[p]) * m, (size_t)h.rcount[p] * m, ncclDouble, p,
                         c->comm, s) != ncclSuccess) { ncclGroupEnd(); return cudaErrorUnknown; }
    }
    return ncclGroupEnd() == ncclSuccess ? cudaSuccess : cudaErrorUnknown;
}

cudaError_t allreduce_sum(double* buf, int64_t count, const mrs_comm* c, cudaStream_t s) {
    return ncclAllReduce(buf, buf, (size_t)count, ncclDouble, ncclSum, c->comm, s) == ncclSuccess
               ? cudaSuccess : cudaErrorUnknown;
}

cudaError_t allgather_inplace(double* buf, int64_t count, const mrs_comm* c, cudaStream_t s) {
    return ncclAllGather(buf + (int64_t)c->rank * count, buf, (size_t)count, ncclDouble, c->comm,
                         s) == ncclSuccess ? cudaSuccess : cudaErrorUnknown;
}

__global__ void __launch_bounds__(kThreads) epilogue_kernel(SolveState* st, const double* vals,
                                                            int Km, int m, int epi,
                                                            const int* guard) {
    if (guard && *guard) return;
    __shared__ double s_v[kMaxK * kMaxM];
    for (int i = threadIdx.x; i < Km; i += blockDim.x) s_v[i] = vals[i];
    __syncthreads();
    run_epilogue(epi, st, s_v, m);
}

cudaError_t launch_epilogue(SolveState* st, const double* vals, int Km, int m, int epi,
                            const int* guard, cudaStream_t s) {
    epilogue_kernel<<<1, kThreads, 0, s>>>(st, vals, Km, m, epi, guard);
    return cudaGetLastError();
}

}  // namespace mrs

using namespace mrs;

extern "C" {

int mrs_comm_unique_id(void* out) {
    if (!out) return MRS_ERR_ARG;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return MRS_ERR_CUDA;
    memcpy(out, &id, sizeof(id));
    return MRS_OK;
}

int mrs_comm_create(const void* id, int32_t rank, int32_t nranks, mrs_comm** out) {
    if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks) return MRS_ERR_ARG;
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof(uid));
    mrs_comm* c = new mrs_comm();
    c->rank = rank;
    c->nranks = nranks;
    if (ncclCommInitRank(&c->comm, nranks, uid, rank) != ncclSuccess) {
        delete c;
        return MRS_ERR_CUDA;
    }
    *out = c;
    return MRS_OK;
}

void mrs_comm_destroy(mrs_comm* c) {
    if (!c) return;
    if (c->comm) ncclCommDestroy(c->comm);
    delete c;
}

}  // extern "C"
