// qgemm_tc.cu — tcgen05 prefill GEMM (placeholder until the tensor-core kernel lands).
#include "common.cuh"
#include "qgemm.cuh"

namespace ifb {
if_status qgemm_tc_launch(if_scheme, const uint8_t*, int64_t, int64_t, const __nv_bfloat16*, int64_t, float*, int,
                          cudaStream_t) {
  return IF_ERR_UNSUPPORTED;
}
}  // namespace ifb
