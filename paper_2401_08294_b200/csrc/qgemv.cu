// qgemv.cu — a4: decode GEMV with fused dequantization:
//     y[b, n] (+)= sum_k W'[n, k] x[b, k],   W' from Eq. 2
//
// Two kernels:
//  * qgemv_q3h64<BT>  — the hot path: Q3H_B64 (0.5 B/weight).  A lane owns one
//    64-weight block column; a warp covers 32 consecutive blocks (a "chunk")
//    of R rows per iteration, each block a single 256-bit streaming load.
//    x is staged once per CTA in shared memory in a pre-transformed,
//    bank-conflict-free layout so that the pair decode of simd.cuh needs 2
//    SASS ops/weight; the per-block scale is factored out:
//        sum_i w'_i x_i = lo * sum(x) + step * sum_i q_i x_i.
//    Partial sums are combined across lanes with shuffles and across chunks in
//    shared memory in a fixed order (deterministic).
//  * qgemv_generic<QT,BS,BT> — every other scheme/batch: one warp per row,
//    lanes stride over blocks, W' = fma(q, step, lo) exactly as Eq. 2, fp32
//    accumulation.  Correct for all schemes; not the tuned path.
#include <algorithm>

#include "common.cuh"
#include "decode_mk.cuh"
#include "qgemm.cuh"
#include "simd.cuh"

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

// ---------------------------------------------------------------------------
// fast Q3H_B64
// ---------------------------------------------------------------------------
struct FastGeom {
  int nb, nchunk, nbp, RG, warps, rows_per_cta;
};

// shared memory: xs  float4 [BT][16][nbp]   {512 x_o(2jj), 512 x_o(2jj+1), xe'(2jj), xe'(2jj+1)}
//                bs  float2 [BT][nbp]       {sum x, sum x_odd} of block b
//                part float  [rows][nchunk][BT]
template <int BT>
__host__ __device__ inline size_t fast_smem_bytes(const FastGeom& g) {
  return (size_t)BT * 16 * g.nbp * 16 + (size_t)BT * g.nbp * 8 + (size_t)g.rows_per_cta * g.nchunk * BT * 4;
}

template <int BT, int R>
__global__ void __launch_bounds__(512) qgemv_q3h64(const uint8_t* __restrict__ W, int N, FastGeom g,
                                                   const float* __restrict__ x, int nbt, float* __restrict__ y,
                                                   int acc_mode) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float4* xs = reinterpret_cast<float4*>(smem_raw);
  float2* bs = reinterpret_cast<float2*>(smem_raw + (size_t)BT * 16 * g.nbp * 16);
  float* part = reinterpret_cast<float*>(smem_raw + (size_t)BT * 16 * g.nbp * 16 + (size_t)BT * g.nbp * 8);
  const int nb = g.nb, nbp = g.nbp, nchunk = g.nchunk;
  const int K = nb * 64;

  // ---- 1. stage transformed x (identity (*) of simd.cuh) ----
  for (int p = threadIdx.x; p < BT * nbp * 32; p += blockDim.x) {
    const int t = p / (nbp * 32), pp = p - t * nbp * 32;
    const int b = pp >> 5, j = pp & 31;
    float xe = 0.f, xo = 0.f;
    if (b < nb && t < nbt) {
      float2 v = __ldg(reinterpret_cast<const float2*>(x + (int64_t)t * K) + pp);
      xe = v.x;
      xo = v.y;
    }
    float* f = reinterpret_cast<float*>(xs + ((size_t)t * 16 + (j >> 1)) * nbp + b);
    f[j & 1] = 512.0f * xo;          // exact scaling
    f[2 + (j & 1)] = fmaf(-11.0f, xo, xe);
  }
  for (int p = threadIdx.x; p < BT * nbp; p += blockDim.x) {
    const int t = p / nbp, b = p - t * nbp;
    float sx = 0.f, sxo = 0.f;
    if (b < nb && t < nbt) {
      const float2* xp = reinterpret_cast<const float2*>(x + (int64_t)t * K + (int64_t)b * 64);
#pragma unroll 8
      for (int i = 0; i < 32; i++) {
        float2 v = __ldg(xp + i);
        sx += v.x + v.y;
        sxo += v.y;
      }
    }
    bs[p] = make_float2(sx, sxo);
  }
  __syncthreads();

  // ---- 2. stream rows ----
  const Q3HConst kc = q3h_const();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = warp % nchunk, grp = warp / nchunk;
  const int b = c * 32 + lane;
  const bool active = b < nb;
  const int row0 = blockIdx.x * g.rows_per_cta;
  const int row1 = min(N, row0 + g.rows_per_cta);
  float2 bsum[BT];
#pragma unroll
  for (int t = 0; t < BT; t++) bsum[t] = bs[t * nbp + b];

  for (int r = row0 + grp * R; r < row1; r += g.RG * R) {
    uint32_t wv[R][8];
#pragma unroll
    for (int i = 0; i < R; i++) {
      if (active && r + i < row1) {
        ldg256_stream(W + ((int64_t)(r + i) * nb + b) * 32, wv[i]);
      } else {
#pragma unroll
        for (int k = 0; k < 8; k++) wv[i][k] = 0u;
      }
    }
    u64 accc[R][BT], accq[R][BT];
#pragma unroll
    for (int i = 0; i < R; i++)
#pragma unroll
      for (int t = 0; t < BT; t++) accc[i][t] = accq[i][t] = 0ull;

#define IFB_PAIR2(JJ)                                                                           \
  {                                                                                             \
    float4 xv[BT];                                                                              \
    _Pragma("unroll") for (int t = 0; t < BT; t++) xv[t] = xs[((size_t)t * 16 + (JJ)) * nbp + b]; \
    _Pragma("unroll") for (int i = 0; i < R; i++) {                                             \
      const uint32_t v0 = q3h_view<2 * (JJ)>(wv[i]);                                            \
      const uint32_t v1 = q3h_view<2 * (JJ) + 1>(wv[i]);                                        \
      const u64 cf = pack2(__uint_as_float(and_or(v0, kc.mask, kc.expo)),                       \
                           __uint_as_float(and_or(v1, kc.mask, kc.expo)));                      \
      const u64 qe = fadd2(ffma2(cf, kc.A2, kc.B2), kc.D2);                                     \
      _Pragma("unroll") for (int t = 0; t < BT; t++) {                                          \
        accc[i][t] = ffma2(cf, pack2(xv[t].x, xv[t].y), accc[i][t]);                            \
        accq[i][t] = ffma2(qe, pack2(xv[t].z, xv[t].w), accq[i][t]);                            \
      }                                                                                         \
    }                                                                                           \
  }
    IFB_PAIR2(0) IFB_PAIR2(1) IFB_PAIR2(2) IFB_PAIR2(3) IFB_PAIR2(4) IFB_PAIR2(5) IFB_PAIR2(6)
    IFB_PAIR2(7) IFB_PAIR2(8) IFB_PAIR2(9) IFB_PAIR2(10) IFB_PAIR2(11) IFB_PAIR2(12)
    IFB_PAIR2(13) IFB_PAIR2(14) IFB_PAIR2(15)
#undef IFB_PAIR2

    // block scale: lo*sum(x) + step*(sum q x), step = (hi-lo)/10 (Eq. 2, D = 10)
#pragma unroll
    for (int i = 0; i < R; i++) {
      const float lo = half_bits_to_float(wv[i][0] & 0xFFFFu);
      const float hi = half_bits_to_float(wv[i][0] >> 16);
      const float step = (hi - lo) * 0.1f;
#pragma unroll
      for (int t = 0; t < BT; t++) {
        const float2 a = unpack2(accc[i][t]);
        const float2 q = unpack2(accq[i][t]);
        const float sq = ((a.x + a.y) - 512.0f * bsum[t].y) + (q.x + q.y);
        float v = fmaf(step, sq, lo * bsum[t].x);
        if (!active) v = 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0 && r + i < row1) part[((r + i - row0) * nchunk + c) * BT + t] = v;
      }
    }
  }
  __syncthreads();

  // ---- 3. combine chunks in fixed order ----
  for (int p = threadIdx.x; p < (row1 - row0) * BT; p += blockDim.x) {
    const int rr = p / BT, t = p - rr * BT;
    if (t >= nbt) continue;
    float s = 0.f;
    for (int cc = 0; cc < nchunk; cc++) s += part[(rr * nchunk + cc) * BT + t];
    float* dst = y + (int64_t)t * N + row0 + rr;
    *dst = acc_mode ? (*dst + s) : s;
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

template <int BT, int R>
static if_status launch_fast(const uint8_t* W, int64_t N, int64_t K, const float* x, int64_t B, float* y,
                             int acc, cudaStream_t st, bool* done) {
  *done = false;
  FastGeom g;
  g.nb = (int)(K / 64);
  g.nchunk = (g.nb + 31) / 32;
  g.nbp = g.nchunk * 32;
  if (g.nchunk > 16) return IF_OK;
  g.RG = std::max(1, 8 / g.nchunk);
  g.warps = g.nchunk * g.RG;
  const int sms = num_sms();
  // ~2 resident CTAs per SM; each CTA gets a contiguous row range
  int64_t ctas = std::min<int64_t>((N + R - 1) / R, (int64_t)sms * 2);
  g.rows_per_cta = (int)((N + ctas - 1) / ctas);
  ctas = (N + g.rows_per_cta - 1) / g.rows_per_cta;
  const size_t smem = fast_smem_bytes<BT>(g);
  if (smem > 200 * 1024) return IF_OK;
  auto kern = qgemv_q3h64<BT, R>;
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(200 * 1024));
    configured = 200 * 1024;
  }
  for (int64_t b0 = 0; b0 < B; b0 += BT) {
    const int nbt = (int)std::min<int64_t>(BT, B - b0);
    kern<<<(unsigned)ctas, g.warps * 32, smem, st>>>(W, (int)N, g, x + b0 * K, nbt, y + b0 * N, acc);
    count_launch();
  }
  *done = true;
  return check_launch("if_qgemv(q3h64)");
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
  if (s.type == IF_Q3H && s.block == 64 && (reinterpret_cast<uintptr_t>(W) & 31u) == 0 && N < (1ll << 31)) {
    bool done = false;
    if_status r;
    if (B == 1 && K <= 65536) {
      // persistent TMA-ring engine (decode_mk.cu), single-phase mode
      static thread_local MkParams P;  // 4 KB of layer pointers; filled per call
      P.mode = MK_MODE_GEMV;
      P.layers = 1;
      P.w[0][0] = W;
      P.x_in = x;
      P.y_out = y;
      P.gemv_N = (int)N;
      P.gemv_K = (int)K;
      P.acc = acc;
      P.dbg = g_mk_dbg;
      r = mk_launch(P, st);
      if (r != IF_ERR_UNSUPPORTED) return r;
    }
    if (B == 1) r = launch_fast<1, 4>(W, N, K, x, B, y, acc, st, &done);
    else if (B == 2) r = launch_fast<2, 2>(W, N, K, x, B, y, acc, st, &done);
    else r = launch_fast<4, 1>(W, N, K, x, B, y, acc, st, &done);
    if (r != IF_OK || done) return r;
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
