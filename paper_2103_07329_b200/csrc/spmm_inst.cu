// spmm_inst.cu -- instantiations of the SpMM family for ONE (value type, op)
// pair, selected at compile time: build.py compiles this file once per pair
// (-DMRS_INST_F32=0/1 -DMRS_INST_OP=0..3) so the eight heavy template sets
// build in parallel.
#include "launch.cuh"

#ifndef MRS_INST_OP
#define MRS_INST_OP 0
#endif
#ifndef MRS_INST_F32
#define MRS_INST_F32 0
#endif

namespace mrs {

#if MRS_INST_F32
template <>
cudaError_t launch_spmm_op_f32<MRS_INST_OP>(const DevCsr& A, const SpArgs& a, int64_t m,
                                            cudaStream_t s, bool generic) {
    return spmm_op<MRS_INST_OP, float>(A, a, m, s, generic);
}
#else
template <>
cudaError_t launch_spmm_op_f64<MRS_INST_OP>(const DevCsr& A, const SpArgs& a, int64_t m,
                                            cudaStream_t s, bool generic) {
    return spmm_op<MRS_INST_OP, double>(A, a, m, s, generic);
}
#endif

}  // namespace mrs
