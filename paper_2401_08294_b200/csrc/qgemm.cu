// qgemm.cu — a5: prefill GEMM with fused dequantization:
//     Y[m, n] = sum_k W'[n, k] X[m, k],  X bf16, W' rounded to bf16, fp32 accumulate.
//
// This file holds the entry point and the tile dequantizer shared by the GEMM
// kernels.  (The tcgen05 kernel lives in qgemm_tc.cu.)
#include <cuda_bf16.h>

#include <algorithm>

#include "common.cuh"
#include "qgemm.cuh"

namespace ifb {

// ---------------------------------------------------------------------------
// SIMT reference-structure kernel: 64x64 output tile per CTA, K step 64.
// Used for shapes the tensor-core kernel does not cover.
// ---------------------------------------------------------------------------
template <int QT, int BS>
__global__ void __launch_bounds__(256) qgemm_simt(const uint8_t* __restrict__ W, int64_t N, int64_t K,
                                                  const __nv_bfloat16* __restrict__ X, int64_t M,
                                                  float* __restrict__ Y, int accumulate) {
  constexpr int D = q_levels(QT);
  constexpr int C = q_width(QT);
  constexpr int NC = q_ncodes(QT, BS);
  constexpr int BB = q_block_bytes(QT, BS);
  constexpr int NW = q_block_words(QT, BS);
  __shared__ float xs[64][65];
  __shared__ float ws[64][65];
  const int64_t m0 = (int64_t)blockIdx.y * 64, n0 = (int64_t)blockIdx.x * 64;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float acc[4][4] = {};
  const int64_t nb = K / BS;
  for (int64_t k0 = 0; k0 < K; k0 += 64) {
    for (int i = threadIdx.x; i < 64 * 64; i += 256) {
      const int r = i >> 6, cc = i & 63;
      const int64_t m = m0 + r;
      xs[r][cc] = (m < M && k0 + cc < K) ? __bfloat162float(X[m * K + k0 + cc]) : 0.f;
    }
    // dequantize 64 rows x 64 k (one or two blocks per row), Eq. 2, rounded to bf16
    for (int i = threadIdx.x; i < 64 * (64 / BS); i += 256) {
      const int r = i / (64 / BS), sub = i % (64 / BS);
      const int64_t n = n0 + r;
      const int64_t kb = k0 / BS + sub;
      if (n < N && kb < nb) {
        uint32_t w[NW + 1];
        load_block_words<BB, NW>(W + (n * nb + kb) * BB, w);
        const float lo = half_bits_to_float(w[0] & 0xFFFFu);
        const float hi = half_bits_to_float(w[0] >> 16);
        const float step = __fdiv_rn(__fsub_rn(hi, lo), (float)D);
#pragma unroll
        for (int j = 0; j < NC; j++) {
          const uint32_t v = get_code<C, NW>(w, j);
          if constexpr (QT == 35) {
            const uint32_t q1 = v / 11u, q2 = v - 11u * q1;
            ws[r][sub * BS + 2 * j] = __bfloat162float(__float2bfloat16(__fmaf_rn((float)q1, step, lo)));
            ws[r][sub * BS + 2 * j + 1] = __bfloat162float(__float2bfloat16(__fmaf_rn((float)q2, step, lo)));
          } else {
            ws[r][sub * BS + j] = __bfloat162float(__float2bfloat16(__fmaf_rn((float)v, step, lo)));
          }
        }
      } else {
        for (int j = 0; j < BS; j++) ws[r][sub * BS + j] = 0.f;
      }
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < 64; kk++) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; i++) {
        a[i] = xs[ty * 4 + i][kk];
        b[i] = ws[tx * 4 + i][kk];
      }
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const int64_t m = m0 + ty * 4 + i, n = n0 + tx * 4 + j;
      if (m < M && n < N) {
        float* d = Y + m * N + n;
        *d = accumulate ? *d + acc[i][j] : acc[i][j];
      }
    }
}

if_status qgemm_simt_launch(if_scheme s, const uint8_t* W, int64_t N, int64_t K, const __nv_bfloat16* X, int64_t M,
                            float* Y, int accumulate, cudaStream_t st) {
  return dispatch_scheme(s, [&]<int QT, int BS>() -> if_status {
    dim3 grid((unsigned)((N + 63) / 64), (unsigned)((M + 63) / 64));
    qgemm_simt<QT, BS><<<grid, 256, 0, st>>>(W, N, K, X, M, Y, accumulate);
    count_launch();
    return check_launch("qgemm_simt");
  });
}

if_status qgemm_impl(const char* fn, if_scheme s, const uint8_t* W, int64_t N, int64_t K, const uint16_t* X,
                     int64_t M, float* Y, int accumulate, cudaStream_t st) {
  if (!scheme_ok(s)) return set_error(IF_ERR_SCHEME, "%s: invalid scheme", fn);
  if (N < 0 || K < 0 || M < 0 || K % s.block)
    return set_error(IF_ERR_SHAPE, "%s: M=%lld N=%lld K=%lld", fn, (long long)M, (long long)N, (long long)K);
  if (M == 0 || N == 0) return IF_OK;
  if (!W || !Y || (K > 0 && !X)) return set_error(IF_ERR_ARG, "%s: null pointer", fn);
  if ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Y) | reinterpret_cast<uintptr_t>(W)) & 15u)
    return set_error(IF_ERR_ARG, "%s: W, X, Y must be 16-byte aligned", fn);
  if (K == 0) {
    if (!accumulate && cudaMemsetAsync(Y, 0, sizeof(float) * M * N, st) != cudaSuccess) return check_launch(fn);
    return IF_OK;
  }
  const __nv_bfloat16* Xb = reinterpret_cast<const __nv_bfloat16*>(X);
  if_status r = qgemm_tc_launch(s, W, N, K, Xb, M, Y, accumulate, st);
  if (r != IF_ERR_UNSUPPORTED) return r;
  return qgemm_simt_launch(s, W, N, K, Xb, M, Y, accumulate, st);
}

}  // namespace ifb

using namespace ifb;

extern "C" if_status if_qgemm(if_scheme s, const uint8_t* W, int64_t N, int64_t K, const uint16_t* X_bf16, int64_t M,
                              float* Y, if_stream_t stream) {
  return qgemm_impl("if_qgemm", s, W, N, K, X_bf16, M, Y, 0, (cudaStream_t)stream);
}
