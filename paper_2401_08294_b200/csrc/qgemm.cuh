// qgemm.cuh — internal interface of the prefill GEMM kernels.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "../../include/if_b200.h"

namespace ifb {
// Y (+)= X W'^T.  Returns IF_ERR_UNSUPPORTED (without launching) for shapes the
// tensor-core kernel does not take.
if_status qgemm_tc_launch(if_scheme s, const uint8_t* W, int64_t N, int64_t K, const __nv_bfloat16* X, int64_t M,
                          float* Y, int accumulate, cudaStream_t st);
// Batched decode on the tensor cores: y[b, n] (+)= sum_k W'[n, k] x[b, k], x fp32
// [B, K] with 1 <= B <= 64 (fp16 hi/lo split in-kernel, W' -> fp16).
if_status qgemv_tc_launch(if_scheme s, const uint8_t* W, int64_t N, int64_t K, const float* x, int64_t B, float* Y,
                          int accumulate, cudaStream_t st);
if_status qgemm_simt_launch(if_scheme s, const uint8_t* W, int64_t N, int64_t K, const __nv_bfloat16* X, int64_t M,
                            float* Y, int accumulate, cudaStream_t st);
if_status qgemm_impl(const char* fn, if_scheme s, const uint8_t* W, int64_t N, int64_t K, const uint16_t* X, int64_t M,
                     float* Y, int accumulate, cudaStream_t st);
}  // namespace ifb
