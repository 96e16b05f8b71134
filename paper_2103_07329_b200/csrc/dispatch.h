// dispatch.h -- host-side launchers shared by the C ABI (capi.cu) and the
// solver plan (solver.cu).  Each picks the template instance for (m, index
// width, value width) and a persistent grid.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/mrsolve_b200.h"
#include "spmm.cuh"
#include "blas.cuh"

namespace mrs {

struct Halo;

struct DevCsr {
    int64_t nrows = 0, ncols = 0, nnz = 0;
    const Halo* halo = nullptr;   // multi-GPU: exchange of the gathered operand before use
    int32_t* slab_base = nullptr; // slab-relative 16-bit column indices (optional)
    int slab_shift = 0;
    int32_t* rp = nullptr;
    void* ci = nullptr;
    void* v = nullptr;
    int ib = 4, vb = 8;
    int32_t* long_rows = nullptr; // rows with > long_thr entries (spmm.cuh long_row_cta)
    int n_long = 0, long_thr = 0;
    int max_row = 0;              // longest row (solver levels; 0 = unknown)
    int variant = 0;              // SpmmVariant chosen for this operator (0 = heuristic)
    // structure facts for the m = 1 stream kernel (stream.cu); unknown = not eligible
    int band = -1;                // max |column - row|
    int blk_max = 0;              // most entries in an aligned block of 256 rows
    bool padded = false;          // >= 64 readable bytes behind ci / v
    bool present() const { return rp != nullptr; }
    // algorithmic bytes of one pass over the CSR arrays
    double bytes() const {
        double sb = slab_base ? (double)(((nrows - 1) >> slab_shift) + 1) * 4.0 : 0.0;
        return (double)nnz * (ib + vb) + (double)(nrows + 1) * 4.0 + sb;
    }
};

// SpMM-family launch (OP = SpOp).  a.rp/ci/vals/nrows are filled from A.
cudaError_t launch_spmm(int op, const DevCsr& A, SpArgs a, int64_t m, cudaStream_t s,
                        bool generic = false);
// m = 1 stream variant (stream.cu): eligibility of one launch, and the launch.
bool spmm_stream_eligible(const DevCsr& A, int64_t m, const SpArgs& a);
cudaError_t launch_spmm_stream(const DevCsr& A, const SpArgs& a, cudaStream_t s);
int64_t spmm_stream_launches();
// Device-side index compression at upload (slab.cu; same rule as core.slab_compress).
int slab_compress_device(const int32_t* rp_dev, const uint32_t* ci32_dev, int64_t nrows, int64_t nnz,
                         int64_t ncols, uint16_t** ci16, int32_t** base, int* shift,
                         int64_t* nslabs);
// Vector-family launch (OP = VecOp).
cudaError_t launch_vec(int op, VArgs a, cudaStream_t s);
// fp32-preconditioner interface kernels (kernels.cu): r -> float b (+ seed), float x -> z
cudaError_t launch_cvt_to32(const double* r, float* b32, int64_t n, int64_t m, int seed_mode,
                            const double* d, double w, float* seed_out, const int* guard,
                            cudaStream_t s);
cudaError_t launch_cvt_from32(const float* x32, double* z, int64_t total, const int* guard,
                              cudaStream_t s);
// Dense coarse solve x = Ainv b for (nc, m) blocks.
cudaError_t launch_dense(const double* T, int64_t n, const double* b, double* x, int64_t m,
                         const int* guard, cudaStream_t s);
cudaError_t launch_coarse(const double* inv, int64_t nc, const double* b, double* x,
                          int64_t m, const int* guard, cudaStream_t s);
void set_coarse_rows(int64_t v);
void set_spmm_long_rows(int64_t v);
void set_spmm_chunk_rows(int64_t v);
void set_spmm_long_split(int64_t v);
void set_spmm_coop(int64_t v);
void set_spmm_pair(int64_t v);
bool dense_mma_enabled();
int64_t loop_unroll();
void set_loop_unroll(int64_t v);
void set_dense_mma(int64_t v);
int64_t spmm_long_split();
int64_t halo_overlap();
// per-operator SpMM variant by measurement (kernels.cu); knob spmm_autotune
// flush: an L2-sized device buffer read before every timed launch (cold
// conditions), or null
// keep: the shape heuristic's variant stays unless the fastest one takes less than
// `keep` of its time (plans: 0.85 -- an isolated launch is only a proxy for the
// operator's cost inside a solve; standalone plugin products: 0.97)
int spmm_tune(const DevCsr& A, const double* x, double* y, int64_t m, cudaStream_t s,
              float* best_us = nullptr, int vp = 0, const double* flush = nullptr,
              int64_t flush_n = 0, float keep = 0.85f);
int64_t spmm_autotune_enabled();
int64_t plan_autotune();
void set_plan_autotune(int64_t v);
void set_spmm_autotune(int64_t v);
void set_spmm_variant(int64_t v);
int64_t spmm_variant();
void set_halo_overlap(int64_t v);
// Gauss-Seidel half-sweep on one thread-block cluster (sgs.cu)
struct SgsArgs;
cudaError_t launch_sgs(const SgsArgs& a, int vb, int ib, cudaStream_t s);
// Grid the reduction kernels use (partials buffer sizing).
int vec_grid(int64_t n, int64_t m);
int spmm_grid(int64_t nrows, int64_t m);
int max_grid();
void set_pdl(int on);
int vec_op_k(int op);   // reduced values per column of a vector op (0 = none)

}  // namespace mrs
