// spmm_f64.cu -- instantiations of the SpMM family for double matrix values
// (separate translation unit: parallel builds).
#include "launch.cuh"

namespace mrs {

cudaError_t launch_spmm_f64(int op, const DevCsr& A, const SpArgs& a, int64_t m, cudaStream_t s,
                            bool generic) {
    switch (op) {
    case OP_SPMV: return spmm_op<OP_SPMV, double>(A, a, m, s, generic);
    case OP_JAC_SWEEP: return spmm_op<OP_JAC_SWEEP, double>(A, a, m, s, generic);
    case OP_CHEB_FIRST: return spmm_op<OP_CHEB_FIRST, double>(A, a, m, s, generic);
    case OP_CHEB_STEP: return spmm_op<OP_CHEB_STEP, double>(A, a, m, s, generic);
    }
    return cudaErrorInvalidValue;
}

}  // namespace mrs
