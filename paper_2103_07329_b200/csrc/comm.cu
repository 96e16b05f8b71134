// comm.cu -- NCCL communicator C ABI, halo exchange, split reductions.
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <vector>

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
        MRS_DCHECK(__ldg(idx + i) >= 0);
        out[e] = x[(int64_t)__ldg(idx + i) * m + c];
    }
}

// ---------------------------------------------------------------------------
// TEST-ONLY loopback transport (see mrs_comm::loop).  Every collective is
//   post my arguments; record "ready" on my stream; host barrier;
//   enqueue my reads of the peers' buffers behind THEIR "ready" events;
//   record "read" on my stream; host barrier; my stream waits for every
//   peer's "read" before it may overwrite what peers read from me.
// Ordering is by stream events only; kernels never wait on each other.
// ---------------------------------------------------------------------------
struct LoopSlot {
    const Halo* h = nullptr;
    double* x = nullptr;          // halo: operand; allreduce / allgather: buffer
    int64_t m = 0, count = 0;
    int op = 0;                   // 1 halo, 2 allreduce, 3 allgather
};

struct LoopGroup {
    int n = 0;
    int refs = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    bool broken = false;
    std::vector<LoopSlot> slot;
    std::vector<cudaEvent_t> ready, read;
    std::vector<double*> tmp;       // allreduce result per rank
    std::vector<int64_t> tmp_cap;
};

static bool loop_barrier(LoopGroup* g) {
    std::unique_lock<std::mutex> lk(g->mu);
    if (g->broken) return false;
    const uint64_t my = g->gen;
    if (++g->arrived == g->n) {
        g->arrived = 0;
        g->gen++;
        g->cv.notify_all();
        return true;
    }
    const bool ok = g->cv.wait_for(lk, std::chrono::seconds(120),
                                   [&] { return g->gen != my || g->broken; });
    if (!ok || g->broken) {     // a rank never arrived: fail every rank
        g->broken = true;
        g->cv.notify_all();
        return false;
    }
    return true;
}

struct LoopSum { const double* src[8]; };

__global__ void loop_sum_kernel(LoopSum a, int n, int64_t count, double* out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        double acc = a.src[0][i];
        for (int q = 1; q < n; ++q) acc = add(acc, a.src[q][i]);   // rank order
        out[i] = acc;
    }
}

static cudaError_t loop_collective(const mrs_comm* c, const LoopSlot& mine, cudaStream_t s) {
    LoopGroup* g = c->loop;
    const int r = c->rank, n = g->n;
    g->slot[r] = mine;
    cudaError_t e = cudaEventRecord(g->ready[r], s);
    if (e != cudaSuccess) return e;
    if (!loop_barrier(g)) return cudaErrorUnknown;
    for (int q = 0; q < n; ++q)
        if (g->slot[q].op != mine.op) return cudaErrorInvalidValue;   // mismatched schedules
    if (mine.op == 1) {                 // halo: pull my imports from each owner's send buffer
        const Halo& h = *mine.h;
        for (int q = 0; q < n; ++q) {
            if (q == r || !h.rcount.size() || h.rcount[q] == 0) continue;
            const Halo& hq = *g->slot[q].h;
            if (hq.scount.size() != (size_t)n || hq.scount[r] != h.rcount[q])
                return cudaErrorInvalidValue;
            if ((e = cudaStreamWaitEvent(s, g->ready[q], 0)) != cudaSuccess) return e;
            e = cudaMemcpyAsync(mine.x + (h.recv_row0 + h.rdisp[q]) * mine.m,
                                hq.sendbuf + (int64_t)hq.sdisp[r] * mine.m,
                                sizeof(double) * (size_t)h.rcount[q] * mine.m,
                                cudaMemcpyDeviceToDevice, s);
            if (e != cudaSuccess) return e;
        }
    } else if (mine.op == 2) {          // allreduce: every rank sums all buffers in rank order
        if (n > 8) return cudaErrorInvalidValue;
        if (g->tmp_cap[r] < mine.count) {
            if (g->tmp[r]) cudaFree(g->tmp[r]);
            if ((e = cudaMalloc(&g->tmp[r], sizeof(double) * mine.count)) != cudaSuccess) return e;
            g->tmp_cap[r] = mine.count;
        }
        LoopSum a{};
        for (int q = 0; q < n; ++q) {
            if (g->slot[q].count != mine.count) return cudaErrorInvalidValue;
            a.src[q] = g->slot[q].x;
            if (q != r && (e = cudaStreamWaitEvent(s, g->ready[q], 0)) != cudaSuccess) return e;
        }
        loop_sum_kernel<<<1, kThreads, 0, s>>>(a, n, mine.count, g->tmp[r]);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    } else {                            // allgather: copy every peer's slice
        for (int q = 0; q < n; ++q) {
            if (q == r) continue;
            if (g->slot[q].count != mine.count) return cudaErrorInvalidValue;
            if ((e = cudaStreamWaitEvent(s, g->ready[q], 0)) != cudaSuccess) return e;
            e = cudaMemcpyAsync(mine.x + q * mine.count, g->slot[q].x + q * mine.count,
                                sizeof(double) * mine.count, cudaMemcpyDeviceToDevice, s);
            if (e != cudaSuccess) return e;
        }
    }
    if ((e = cudaEventRecord(g->read[r], s)) != cudaSuccess) return e;
    if (!loop_barrier(g)) return cudaErrorUnknown;
    for (int q = 0; q < n; ++q)
        if (q != r && (e = cudaStreamWaitEvent(s, g->read[q], 0)) != cudaSuccess) return e;
    if (mine.op == 2)
        e = cudaMemcpyAsync(mine.x, g->tmp[r], sizeof(double) * mine.count,
                            cudaMemcpyDeviceToDevice, s);
    return e;
}

cudaError_t halo_pack(const Halo& h, const double* x, int64_t m, const int* guard, cudaStream_t s) {
    if (!h.nsend) return cudaSuccess;
    const int64_t total = (int64_t)h.nsend * m;
    int g = (int)((total + kThreads - 1) / kThreads);
    if (g > max_grid()) g = max_grid();
    pack_kernel<<<g, kThreads, 0, s>>>(x, h.send_idx, h.nsend, (int)m, h.sendbuf, guard);
    return cudaGetLastError();
}

cudaError_t halo_transfer(const Halo& h, double* x, int64_t m, const mrs_comm* c, cudaStream_t s) {
    if (c->loop) {
        LoopSlot sl;
        sl.h = &h; sl.x = x; sl.m = m; sl.op = 1;
        return loop_collective(c, sl, s);
    }
    if (!h.active()) return cudaSuccess;
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

cudaError_t halo_exchange(const Halo& h, double* x, int64_t m, const mrs_comm* c, const int* guard,
                          cudaStream_t s) {
    if (!c->loop && !h.active()) return cudaSuccess;
    cudaError_t e = halo_pack(h, x, m, guard, s);
    if (e != cudaSuccess) return e;
    return halo_transfer(h, x, m, c, s);
}

cudaError_t allreduce_sum(double* buf, int64_t count, const mrs_comm* c, cudaStream_t s) {
    if (c->loop) {
        LoopSlot sl;
        sl.x = buf; sl.count = count; sl.op = 2;
        return loop_collective(c, sl, s);
    }
    return ncclAllReduce(buf, buf, (size_t)count, ncclDouble, ncclSum, c->comm, s) == ncclSuccess
               ? cudaSuccess : cudaErrorUnknown;
}

cudaError_t allgather_inplace(double* buf, int64_t count, const mrs_comm* c, cudaStream_t s) {
    if (c->loop) {
        LoopSlot sl;
        sl.x = buf; sl.count = count; sl.op = 3;
        return loop_collective(c, sl, s);
    }
    return ncclAllGather(buf + (int64_t)c->rank * count, buf, (size_t)count, ncclDouble, c->comm,
                         s) == ncclSuccess ? cudaSuccess : cudaErrorUnknown;
}

__global__ void __launch_bounds__(kThreads) epilogue_kernel(SolveState* st, const double* vals,
                                                            int Km, int m, int epi,
                                                            const int* guard, int nsets) {
    if (guard && *guard) return;
    __shared__ double s_v[kMaxK * kMaxM];
    for (int i = threadIdx.x; i < Km; i += blockDim.x) {
        double v = vals[i];
        for (int k = 1; k < nsets; ++k) v = add(v, vals[(int64_t)k * Km + i]);
        s_v[i] = v;
    }
    __syncthreads();
    run_epilogue(epi, st, s_v, m);
}

cudaError_t launch_epilogue(SolveState* st, const double* vals, int Km, int m, int epi,
                            const int* guard, cudaStream_t s, int nsets) {
    epilogue_kernel<<<1, kThreads, 0, s>>>(st, vals, Km, m, epi, guard, nsets);
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
    if (c->loop) {
        LoopGroup* g = c->loop;
        bool last;
        {
            std::lock_guard<std::mutex> lk(g->mu);
            last = --g->refs == 0;
        }
        if (last) {
            for (int q = 0; q < g->n; ++q) {
                cudaEventDestroy(g->ready[q]);
                cudaEventDestroy(g->read[q]);
                if (g->tmp[q]) cudaFree(g->tmp[q]);
            }
            delete g;
        }
    }
    delete c;
}

// TEST-ONLY: nranks communicators joined by the in-process loopback
// transport (mrs_comm::loop); out[r] is rank r's.  Every rank's plan must be
// driven by its own host thread and stream (exec mode eager).
int mrs_comm_create_loopback(int32_t nranks, mrs_comm** out) {
    if (!out || nranks < 1 || nranks > 8) return MRS_ERR_ARG;
    LoopGroup* g = new LoopGroup();
    g->n = nranks;
    g->refs = nranks;
    g->slot.resize(nranks);
    g->ready.resize(nranks);
    g->read.resize(nranks);
    g->tmp.assign(nranks, nullptr);
    g->tmp_cap.assign(nranks, 0);
    for (int q = 0; q < nranks; ++q) {
        if (cudaEventCreateWithFlags(&g->ready[q], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&g->read[q], cudaEventDisableTiming) != cudaSuccess)
            return MRS_ERR_CUDA;
        mrs_comm* c = new mrs_comm();
        c->rank = q;
        c->nranks = nranks;
        c->loop = g;
        out[q] = c;
    }
    return MRS_OK;
}

}  // extern "C"
