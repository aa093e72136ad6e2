// qgemm.cuh — internal interface of the prefill GEMM kernels.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "../../include/if_b200.h"

namespace ifb {
// Y (+)= X W'^T.  Returns IF_ERR_UNSUPPORTED (without launching) for shapes the
// tensor-core kernel does not take.
if_status qgemm_tc_launch(if_scheme s, const uint8_t* W, int64_t N, int64_t K, const __nv_bfloat16* X, int64_t M,
                          float* Y, int accumulate, cudaStream_t st);
// Batched decode on the tensor cores: y[b, n] (+)= sum_k W'[n, k] x[b, k], x fp32
// [B, K] with 1 <= B <= 64 (fp16 hi/lo split, W' -> fp16).  x2_scratch (nullable,
// device, >= 2 * 64 * K * 2 bytes): split x once into it instead of in every CTA.
// x2_ready: the caller already wrote the split into x2_scratch (layout [2 bp, K] fp16:
// rows [0, bp) hi, [bp, 2 bp) lo, zero rows for tokens >= B; bp = tc_bpad(B)).
if_status qgemv_tc_launch(if_scheme s, const uint8_t* W, int64_t N, int64_t K, const float* x, int64_t B, float* Y,
                          int accumulate, cudaStream_t st, void* x2_scratch = nullptr, size_t x2_bytes = 0,
                          int x2_ready = 0);
// Q3H_B64, 2 <= B <= 32: warp-level mma.sync with the decode in registers (qgemv_ms.cu)
// fused batched decode chain (qgemv_ms.cu): 4 launches per layer + 1, T in [2, 16]
struct MsChainLayer {
  const uint8_t *wqkv, *wo, *wgu, *wdown;
};
size_t ms_chain_ws_bytes(int64_t d, int64_t nq, int64_t lf);
// attention step of a KV-cache chain: layer l, ctx record buffer, token tiles per block
typedef if_status (*MsAttnFn)(void* ctx, int layer, uint8_t* rec_ctx, int nt);
if_status ms_chain_run(const MsChainLayer* layers, int nlayers, int64_t d, int64_t lh, int64_t lkv, int64_t hd,
                       int64_t lf, int per, int64_t T, float* h, float* last_qkv, void* ws, cudaStream_t st,
                       MsAttnFn attn = nullptr, void* actx = nullptr, float* qkv_buf = nullptr);
if_status qgemv_ms_launch(if_scheme s, const uint8_t* W, int64_t N, int64_t K, const __half* x2, const float* sc,
                          int64_t B, float* y, int accumulate, cudaStream_t st);
// if_qgemv / if_qgemv_acc with optional tensor-core scratch (the stack's workspace)
if_status qgemv_dispatch(const char* fn, if_scheme s, const uint8_t* W, int64_t N, int64_t K, const float* x,
                         int64_t B, float* y, int acc, cudaStream_t st, void* x2_scratch, size_t x2_bytes,
                         int x2_ready = 0);
// token rows of the fp16 hi/lo split (and of the decode UMMA N/2): B rounded up to 8/16/32/64
__host__ __device__ constexpr int tc_bpad(int B) { return B <= 8 ? 8 : B <= 16 ? 16 : B <= 32 ? 32 : 64; }
if_status qgemm_simt_launch(if_scheme s, const uint8_t* W, int64_t N, int64_t K, const __nv_bfloat16* X, int64_t M,
                            float* Y, int accumulate, cudaStream_t st);
if_status qgemm_impl(const char* fn, if_scheme s, const uint8_t* W, int64_t N, int64_t K, const uint16_t* X, int64_t M,
                     float* Y, int accumulate, cudaStream_t st);
}  // namespace ifb
