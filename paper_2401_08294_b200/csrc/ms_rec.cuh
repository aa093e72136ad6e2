// ms_rec.cuh — fragment records of the fused batched decode chain (qgemv_ms.cu): the
// input of one chain GEMV, written by the producer of that input (the previous phase's
// split-K owner, or the KV attention merge) in the mma.sync B-fragment order.
//
// Record of (64-block kb, token tile t), FR_REC bytes, kb-major (a K-range is contiguous):
//   [0, 2048)    fragments uint4 [hi/lo][q][32 lanes] (lane 4 g + c = token g of the tile,
//                values x[16c, 16c+16) of the block, permuted as qgemv_ms.cu describes)
//   [2048, 2112) float4 [cq] = {5 So(2cq), 5 So(2cq+1), S(2cq), S(2cq+1)} (unscaled sums)
//   [2112, 2176) float4 [cq] = {2^-k(2cq), 2^-k(2cq+1), 0, 0}
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

#include "common.cuh"

namespace ifb {

constexpr int FR_REC = 2176;

__device__ __forceinline__ uint32_t ms_h2u(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }

// One item = (token tok, 16 values x[16c, 16c+16) of one 64-block); the four items of a
// (token, block) sit in adjacent lanes c = lane & 3 (all 32 lanes call, `ok` masks).
__device__ __forceinline__ void ms_put_item(uint8_t* rec, int tok, int c, const float (&x)[16], bool ok) {
  float amax = 0.f, s = 0.f, so = 0.f;
#pragma unroll
  for (int i = 0; i < 16; i++) amax = fmaxf(amax, fabsf(x[i]));
#pragma unroll
  for (int i = 0; i < 8; i++) {
    s += x[2 * i] + x[2 * i + 1];
    so += x[2 * i + 1];
  }
  amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 1));
  amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 2));
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  so += __shfl_xor_sync(0xffffffffu, so, 1);
  so += __shfl_xor_sync(0xffffffffu, so, 2);
  if (!ok) return;
  const int k = xsplit_k(amax) - 4;  // |x| 2^k < 2^11: |x_e - 11 x_o| 2^k < 24576
  const float sig = pow2f(k);
  float fv[16];
#pragma unroll
  for (int m = 0; m < 4; m++) {
    const int a = (m & 1) + 4 * (m >> 1), b = a + 2;
    fv[4 * m + 0] = 0.25f * sig * x[2 * a + 1];
    fv[4 * m + 1] = sig * x[2 * b + 1];
    fv[4 * m + 2] = sig * fmaf(-11.f, x[2 * a + 1], x[2 * a]);
    fv[4 * m + 3] = sig * fmaf(-11.f, x[2 * b + 1], x[2 * b]);
  }
  uint32_t fh[8], fl[8];
#pragma unroll
  for (int i = 0; i < 8; i++) {
    const __half2 hh = __floats2half2_rn(fv[2 * i], fv[2 * i + 1]);
    const float2 hf = __half22float2(hh);
    fh[i] = ms_h2u(hh);
    fl[i] = ms_h2u(__floats2half2_rn(fv[2 * i] - hf.x, fv[2 * i + 1] - hf.y));
  }
  const int fl_lane = 4 * (tok & 7) + c;
  uint4* f = reinterpret_cast<uint4*>(rec) + fl_lane;
  f[0] = make_uint4(fh[0], fh[1], fh[2], fh[3]);
  f[32] = make_uint4(fh[4], fh[5], fh[6], fh[7]);
  f[64] = make_uint4(fl[0], fl[1], fl[2], fl[3]);
  f[96] = make_uint4(fl[4], fl[5], fl[6], fl[7]);
  if (c == 0) {
    float* sp = reinterpret_cast<float*>(rec + 2048) + 4 * ((tok >> 1) & 3);
    const int e = tok & 1;
    sp[e] = 5.f * so;
    sp[2 + e] = s;
    sp[16 + e] = pow2f(-k);
    sp[18 + e] = 0.f;
  }
}

}  // namespace ifb
