// spgemm.h -- Galerkin triple product of the AMG setup on the GPU (spgemm.cu).
//
// SURVEY 8(f) rank 2 (AMG setup on the GPU), the dominant setup phase: the
// coarse operator A_c = (R A) P of every level (reference src/amg.py:185-196,
// scipy csr_matmat).  The arithmetic of the reference is reproduced exactly --
// for every output entry the products are added in the (jj, kk) traversal order
// of scipy's SMMP kernel with separately rounded multiply and add, exact zeros
// are dropped, and the intermediate R A keeps scipy's row emission order
// (reverse first touch), which fixes the summation order of the second product
// -- so the hierarchy is bitwise the one the host path (amg_setup.cpp matmat)
// and the reference build.
#pragma once

#include <cstdint>
#include <vector>

namespace mrs {

struct HostCsrView {
    int64_t nrows, ncols;
    const int64_t* rp;
    const int64_t* ci;
    const double* v;
};

// A_c = (R A) P with rows sorted by column.  Returns false when no GPU is usable
// (or on any CUDA error / index overflow): the caller then runs the host path.
bool galerkin_gpu(const HostCsrView& R, const HostCsrView& A, const HostCsrView& P,
                  std::vector<int64_t>& rp, std::vector<int64_t>& ci, std::vector<double>& v);

// Knob (mrs_set_option "setup_gpu"; env MRS_SETUP_GPU): 1 = use the GPU when present.
void set_setup_gpu(int64_t v);
int64_t setup_gpu();
// products computed on the GPU so far (diagnostics)
int64_t galerkin_gpu_count();

}  // namespace mrs
