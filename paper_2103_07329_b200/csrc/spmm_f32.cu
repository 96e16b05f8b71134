// spmm_f32.cu -- instantiations of the SpMM family for float matrix values
// (separate translation unit: parallel builds).
#include "launch.cuh"

namespace mrs {

cudaError_t launch_spmm_f32(int op, const DevCsr& A, const SpArgs& a, int64_t m, cudaStream_t s,
                            bool generic) {
    switch (op) {
    case OP_SPMV: return spmm_op<OP_SPMV, float>(A, a, m, s, generic);
    case OP_JAC_SWEEP: return spmm_op<OP_JAC_SWEEP, float>(A, a, m, s, generic);
    case OP_CHEB_FIRST: return spmm_op<OP_CHEB_FIRST, float>(A, a, m, s, generic);
    case OP_CHEB_STEP: return spmm_op<OP_CHEB_STEP, float>(A, a, m, s, generic);
    }
    return cudaErrorInvalidValue;
}

}  // namespace mrs
