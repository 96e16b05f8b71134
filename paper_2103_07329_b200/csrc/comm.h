// comm.h -- multi-GPU plumbing of the solve path: NCCL communicator, halo
// plans (reference ExchangePlan, src/parallel.py:259-300) and the exchange /
// split-reduction launches the plan schedules.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

#include <vector>

#include "reduce.cuh"

namespace mrs { struct LoopGroup; }

struct mrs_comm {
    ncclComm_t comm = nullptr;
    int rank = 0, nranks = 1;
    // TEST-ONLY loopback transport (mrs_comm_create_loopback): the ranks are
    // plans of ONE process on ONE device, each driven by its own host thread
    // and stream; collectives are host barriers + stream-event ordering +
    // device-to-device copies (no kernel ever waits on another).  Never
    // created by the product's GpuTeam, which always uses NCCL.
    mrs::LoopGroup* loop = nullptr;
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
    // rows of the CONSUMER block that read no halo column: [ilo, ihi) (the
    // longest such run; ihi <= ilo: none).  The product of those rows can run
    // while the exchange is in flight (blas2.py:62-69 does
    // the diagonal block first, off-diagonal blocks after the halo).
    int64_t ilo = 0, ihi = 0;
    bool active() const { return nsend > 0 || nrecv > 0; }
};

// pack + grouped ncclSend/ncclRecv of operand x (m columns)
cudaError_t halo_exchange(const Halo& h, double* x, int64_t m, const mrs_comm* c, const int* guard,
                          cudaStream_t s);
// the two halves of halo_exchange: pack my exported rows (on the compute
// stream), then move them (on a communication stream, overlapping compute)
cudaError_t halo_pack(const Halo& h, const double* x, int64_t m, const int* guard, cudaStream_t s);
cudaError_t halo_transfer(const Halo& h, double* x, int64_t m, const mrs_comm* c, cudaStream_t s);
// in-place sum over ranks of `count` doubles
cudaError_t allreduce_sum(double* buf, int64_t count, const mrs_comm* c, cudaStream_t s);
// in-place allgather: rank r's slice is buf[r*count, (r+1)*count)
cudaError_t allgather_inplace(double* buf, int64_t count, const mrs_comm* c, cudaStream_t s);
// run a reduction epilogue on already-reduced values (1 CTA); nsets > 1: the
// values are nsets consecutive partial sets of Km values, summed in set order
// first (split launches)
cudaError_t launch_epilogue(SolveState* st, const double* vals, int Km, int m, int epi,
                            const int* guard, cudaStream_t s, int nsets = 1);

}  // namespace mrs
