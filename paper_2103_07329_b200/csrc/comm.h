// comm.h -- multi-GPU plumbing of the solve path: NCCL communicator, halo
// plans (reference ExchangePlan, src/parallel.py:259-300) and the exchange /
// split-reduction launches the plan schedules.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

#include <vector>

#include "reduce.cuh"

struct mrs_comm {
    ncclComm_t comm = nullptr;
    int rank = 0, nranks = 1;
};

namespace mrs {

// One operand exchange: the rows of MY local vector other ranks import, and
// the rows I import, received straight into the halo segment
// [recv_row0, recv_row0 + nrecv) of the operand (halo ordered by owner, then
// global id -- owners hold contiguous row ranges).
struct Halo {
    int32_t* send_idx = nullptr;      // device, nsend local row indices grouped by peer
    double* sendbuf = nullptr;        // device, nsend * m
    int nsend = 0, nrecv = 0;
    std::vector<int> scount, sdisp, rcount, rdisp;   // rows per peer
    int64_t recv_row0 = 0;
    bool active() const { return nsend > 0 || nrecv > 0; }
};

// pack + grouped ncclSend/ncclRecv of operand x (m columns)
cudaError_t halo_exchange(const Halo& h, double* x, int64_t m, const mrs_comm* c, const int* guard,
                          cudaStream_t s);
// in-place sum over ranks of `count` doubles
cudaError_t allreduce_sum(double* buf, int64_t count, const mrs_comm* c, cudaStream_t s);
// in-place allgather: rank r's slice is buf[r*count, (r+1)*count)
cudaError_t allgather_inplace(double* buf, int64_t count, const mrs_comm* c, cudaStream_t s);
// run a reduction epilogue on already-reduced values (1 CTA)
cudaError_t launch_epilogue(SolveState* st, const double* vals, int Km, int m, int epi,
                            const int* guard, cudaStream_t s);

}  // namespace mrs
