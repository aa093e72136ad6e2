// qgemv.cu — a4: decode GEMV with fused dequantization:
//     y[b, n] (+)= sum_k W'[n, k] x[b, k],   W' from Eq. 2
//
// Entry points if_qgemv / if_qgemv_acc and their dispatch:
//  * B = 1, Q3H_B64: the persistent TMA-ring engine (decode_mk.cu, single-phase mode);
//  * B >= 2: the tcgen05 batched-decode kernel (qgemm_tc.cu);
//  * anything those cannot take (other schemes at B = 1, unaligned rows, K > 65536):
//    qgemv_generic<QT,BS,BT> below -- one warp per row, lanes stride over blocks,
//    W' = fma(q, step, lo) exactly as Eq. 2, fp32 accumulation.  Correct for all
//    schemes; not a tuned path.
#include <algorithm>

#include "common.cuh"
#include "decode_mk.cuh"
#include "qgemm.cuh"

namespace ifb {

// ---------------------------------------------------------------------------
// generic
// ---------------------------------------------------------------------------
template <int QT, int BS, int BT>
__global__ void __launch_bounds__(256) qgemv_generic(const uint8_t* __restrict__ W, int64_t N, int64_t K,
                                                     const float* __restrict__ x, int B,
                                                     float* __restrict__ y, int acc_mode) {
  constexpr int D = q_levels(QT);
  constexpr int C = q_width(QT);
  constexpr int NC = q_ncodes(QT, BS);
  constexpr int BB = q_block_bytes(QT, BS);
  constexpr int NW = q_block_words(QT, BS);
  const int lane = threadIdx.x & 31;
  const int64_t nb = K / BS;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t n = warp; n < N; n += nwarps) {
    for (int b0 = 0; b0 < B; b0 += BT) {
      float acc[BT];
#pragma unroll
      for (int t = 0; t < BT; t++) acc[t] = 0.f;
      for (int64_t blk = lane; blk < nb; blk += 32) {
        uint32_t w[NW + 1];
        load_block_words<BB, NW>(W + (n * nb + blk) * BB, w);
        const float lo = half_bits_to_float(w[0] & 0xFFFFu);
        const float hi = half_bits_to_float(w[0] >> 16);
        const float step = __fdiv_rn(__fsub_rn(hi, lo), (float)D);
        float wp[BS];
#pragma unroll
        for (int j = 0; j < NC; j++) {
          const uint32_t v = get_code<C, NW>(w, j);
          if constexpr (QT == 35) {
            const uint32_t q1 = v / 11u, q2 = v - 11u * q1;
            wp[2 * j] = __fmaf_rn((float)q1, step, lo);
            wp[2 * j + 1] = __fmaf_rn((float)q2, step, lo);
          } else {
            wp[j] = __fmaf_rn((float)v, step, lo);
          }
        }
#pragma unroll
        for (int t = 0; t < BT; t++) {
          if (b0 + t < B) {
            const float4* xp = reinterpret_cast<const float4*>(x + (int64_t)(b0 + t) * K + blk * BS);
            float s = 0.f;
#pragma unroll
            for (int i = 0; i < BS / 4; i++) {
              float4 xv = __ldg(xp + i);
              s = fmaf(wp[4 * i], xv.x, s);
              s = fmaf(wp[4 * i + 1], xv.y, s);
              s = fmaf(wp[4 * i + 2], xv.z, s);
              s = fmaf(wp[4 * i + 3], xv.w, s);
            }
            acc[t] += s;
          }
        }
      }
#pragma unroll
      for (int t = 0; t < BT; t++) {
        float v = acc[t];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0 && b0 + t < B) {
          float* dst = y + (int64_t)(b0 + t) * N + n;
          *dst = acc_mode ? (*dst + v) : v;
        }
      }
    }
  }
}

static int g_num_sms = 0;
unsigned long long* g_mk_dbg = nullptr;
static int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

template <int BT>
static void launch_generic_t(if_scheme s, const uint8_t* W, int64_t N, int64_t K, const float* x, int64_t B,
                             float* y, int acc, cudaStream_t st) {
  dispatch_scheme(s, [&]<int QT, int BS>() -> if_status {
    const int sms = num_sms();
    int64_t blocks = std::min<int64_t>((N + 7) / 8, (int64_t)sms * 8);
    if (blocks < 1) blocks = 1;
    qgemv_generic<QT, BS, BT><<<(unsigned)blocks, 256, 0, st>>>(W, N, K, x, (int)B, y, acc);
    count_launch();
    return IF_OK;
  });
}

static if_status qgemv_impl(const char* fn, if_scheme s, const uint8_t* W, int64_t N, int64_t K,
                            const float* x, int64_t B, float* y, int acc, if_stream_t stream,
                            void* x2_scratch = nullptr, size_t x2_bytes = 0, int x2_ready = 0) {
  if (!scheme_ok(s)) return set_error(IF_ERR_SCHEME, "%s: invalid scheme type=%d block=%d", fn, s.type, s.block);
  if (N < 0 || K < 0 || K % s.block) return set_error(IF_ERR_SHAPE, "%s: N=%lld K=%lld", fn, (long long)N, (long long)K);
  if (B < 1 || B > 64) return set_error(IF_ERR_ARG, "%s: B=%lld outside 1..64", fn, (long long)B);
  if (N == 0) return IF_OK;
  if (!W || !y || (K > 0 && !x)) return set_error(IF_ERR_ARG, "%s: null pointer", fn);
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y) | reinterpret_cast<uintptr_t>(W)) & 15u)
    return set_error(IF_ERR_ARG, "%s: W, x, y must be 16-byte aligned", fn);
  cudaStream_t st = (cudaStream_t)stream;
  if (K == 0) {  // empty reduction: y = 0 (or unchanged when accumulating)
    if (!acc) {
      if (cudaMemsetAsync(y, 0, sizeof(float) * N * B, st) != cudaSuccess) return check_launch(fn);
    }
    return IF_OK;
  }
  if (B >= 2) {
    // batched decode: the tensor cores (fp16 W', fp16 hi/lo x), weights streamed once
    if_status r = qgemv_tc_launch(s, W, N, K, x, B, y, acc, st, x2_scratch, x2_bytes, x2_ready);
    if (r != IF_ERR_UNSUPPORTED) return r;
  }
  // batch 1: the persistent TMA-ring engine for every scheme but Q3H_B32 (18-byte blocks)
  if (!(s.type == IF_Q3H && s.block == 32) && (reinterpret_cast<uintptr_t>(W) & 31u) == 0 && N < (1ll << 31)) {
    if (B == 1 && K <= 65536) {
      // persistent TMA-ring engine (decode_mk.cu), single-phase mode
      static thread_local MkParams P;  // 4 KB of layer pointers; filled per call
      P.mode = MK_MODE_GEMV;
      P.qt = s.type;
      P.bs = s.block;
      P.tp = 1;
      P.grid = 0;
      P.layers = 1;
      P.w[0][0] = W;
      P.x_in = x;
      P.y_out = y;
      P.gemv_N = (int)N;
      P.gemv_K = (int)K;
      P.acc = acc;
      P.dbg = g_mk_dbg;
      const if_status r = mk_launch(P, st);
      if (r != IF_ERR_UNSUPPORTED) return r;
    }
  }
  if (B == 1) launch_generic_t<1>(s, W, N, K, x, B, y, acc, st);
  else if (B <= 4) launch_generic_t<4>(s, W, N, K, x, B, y, acc, st);
  else launch_generic_t<8>(s, W, N, K, x, B, y, acc, st);
  return check_launch(fn);
}

if_status qgemv_dispatch(const char* fn, if_scheme s, const uint8_t* W, int64_t N, int64_t K, const float* x,
                         int64_t B, float* y, int acc, cudaStream_t st, void* x2_scratch, size_t x2_bytes,
                         int x2_ready) {
  return qgemv_impl(fn, s, W, N, K, x, B, y, acc, (if_stream_t)st, x2_scratch, x2_bytes, x2_ready);
}

}  // namespace ifb

using namespace ifb;

// instrumentation hook (not in the public header): per-CTA phase timestamps
extern "C" void ifx_set_mk_debug(unsigned long long* buf) { ifb::g_mk_dbg = buf; }

extern "C" if_status if_qgemv(if_scheme s, const uint8_t* W, int64_t N, int64_t K, const float* x, int64_t B,
                              float* y, if_stream_t stream) {
  return qgemv_impl("if_qgemv", s, W, N, K, x, B, y, 0, stream);
}

extern "C" if_status if_qgemv_acc(if_scheme s, const uint8_t* W, int64_t N, int64_t K, const float* x,
                                  int64_t B, float* y, if_stream_t stream) {
  return qgemv_impl("if_qgemv_acc", s, W, N, K, x, B, y, 1, stream);
}
