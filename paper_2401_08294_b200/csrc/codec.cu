// codec.cu — a1/a2/a3 on the GPU: block quantization (Eq. 1; the
// 3.5-bit variant P:120-127), the 7-bit pair code, dequantization
// (Eq. 2), plus the synthetic input generator.
//
// Bit-exactness discipline (Q1-Q7): every float op is an explicit
// IEEE round-to-nearest intrinsic (__fsub_rn/__fdiv_rn/__fmul_rn/__fmaf_rn),
// directed fp16 conversion (__float2half_rd/_ru -> F2F.F16.F32.RM/RP),
// roundf = round half away from zero.  Built without --use_fast_math.
//
// These kernels are HBM-bound and off the decode hot path (PTQ is offline,
// P:97); one thread owns one block: contiguous 128/256-byte float4 reads, the
// whole block in registers, codes packed into registers, word stores.
#include "common.cuh"

namespace ifb {

// ---------------------------------------------------------------------------
// synthetic generator (same counter-based generator as synth/__init__.py)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void synth_kernel(uint64_t base, float c, float* __restrict__ out, int64_t n, int64_t offset) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    uint64_t h = splitmix64(base ^ ((uint64_t)(offset + i) * 0xD1B54A32D192ED03ull));
    int32_t s = (int32_t)(h & 0xFFFF) + (int32_t)((h >> 16) & 0xFFFF) + (int32_t)((h >> 32) & 0xFFFF) +
                (int32_t)((h >> 48) & 0xFFFF) - 131070;
    out[i] = __fmul_rn((float)s, c);
  }
}

// ---------------------------------------------------------------------------
// quantize: one thread per block
// ---------------------------------------------------------------------------
template <int QT, int BS>
__global__ void __launch_bounds__(128) quantize_kernel(const float* __restrict__ W, int64_t nblocks,
                                                       uint8_t* __restrict__ out, int32_t* dev_status) {
  constexpr int D = q_levels(QT);
  constexpr int C = q_width(QT);
  constexpr int NC = q_ncodes(QT, BS);
  constexpr int BB = q_block_bytes(QT, BS);
  constexpr int NCW = (q_code_bytes(QT, BS) + 3) / 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t blk = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; blk < nblocks; blk += stride) {
    // blocks of a row-major [N,K] tensor with K % BS == 0 are contiguous runs
    const float4* src = reinterpret_cast<const float4*>(W + blk * BS);
    float w[BS];
#pragma unroll
    for (int i = 0; i < BS / 4; i++) {
      float4 v = __ldg(src + i);
      w[4 * i] = v.x;
      w[4 * i + 1] = v.y;
      w[4 * i + 2] = v.z;
      w[4 * i + 3] = v.w;
    }
    // step 1-2: finiteness, min/max, -0 -> +0 (Q7, Q8)
    bool bad = false;
    float m = w[0], M = w[0];
#pragma unroll
    for (int i = 0; i < BS; i++) {
      bad |= !isfinite(w[i]);
      m = fminf(m, w[i]);
      M = fmaxf(M, w[i]);
    }
    m = __fadd_rn(m, 0.0f);
    M = __fadd_rn(M, 0.0f);
    // step 3: two FP16 numbers, directed rounding (Q3)
    const uint32_t lo16 = __half_as_ushort(__float2half_rd(m));
    const uint32_t hi16 = __half_as_ushort(__float2half_ru(M));
    bad |= ((lo16 & 0x7C00u) == 0x7C00u) || ((hi16 & 0x7C00u) == 0x7C00u);
    if (bad) report_status(dev_status, IF_ERR_INPUT);
    const float lo = half_bits_to_float(lo16);
    const float hi = half_bits_to_float(hi16);
    const float r = __fsub_rn(hi, lo);
    // step 4: q = Round((w - min)/(max - min) * D)  (Eq. 1 / P:122)
    uint32_t q[BS];
#pragma unroll
    for (int i = 0; i < BS; i++) {
      float t = __fmul_rn(__fdiv_rn(__fsub_rn(w[i], lo), r), (float)D);
      float rq = roundf(t);  // Q1: half away from zero
      rq = fminf(fmaxf(rq, 0.0f), (float)D);
      q[i] = (r == 0.0f) ? 0u : (uint32_t)rq;  // Q6
    }
    // step 5: codes, tight LSB-first bit packing (Q11); Q3H pair code
    uint32_t cw[NCW + 1];
#pragma unroll
    for (int i = 0; i <= NCW; i++) cw[i] = 0;
#pragma unroll
    for (int j = 0; j < NC; j++) {
      const uint32_t v = (QT == 35) ? q[2 * j] * 11u + q[2 * j + 1] : q[j];
      const int bit = j * C;
      cw[bit >> 5] |= v << (bit & 31);
      if ((bit & 31) + C > 32) cw[(bit >> 5) + 1] |= v >> (32 - (bit & 31));
    }
    uint8_t* dst = out + blk * BB;
    const uint32_t hdr = lo16 | (hi16 << 16);  // [lo16 LE][hi16 LE] (Q12)
    if constexpr (BB % 4 == 0) {
      uint32_t* d32 = reinterpret_cast<uint32_t*>(dst);
      d32[0] = hdr;
#pragma unroll
      for (int i = 0; i < NCW; i++) d32[1 + i] = cw[i];
    } else {
      uint16_t* d16 = reinterpret_cast<uint16_t*>(dst);  // BB is even for every scheme
      d16[0] = (uint16_t)lo16;
      d16[1] = (uint16_t)hi16;
#pragma unroll
      for (int i = 0; i < (BB - 4) / 2; i++) d16[2 + i] = (uint16_t)(cw[i >> 1] >> ((i & 1) * 16));
    }
  }
}

// ---------------------------------------------------------------------------
// dequantize: one thread per block (Eq. 2 as fma32(q, r/D, lo), Q5)
// ---------------------------------------------------------------------------
template <int QT, int BS>
__global__ void __launch_bounds__(128) dequantize_kernel(const uint8_t* __restrict__ packed, int64_t nblocks,
                                                         float* __restrict__ out, int32_t* dev_status) {
  constexpr int D = q_levels(QT);
  constexpr int C = q_width(QT);
  constexpr int NC = q_ncodes(QT, BS);
  constexpr int BB = q_block_bytes(QT, BS);
  constexpr int NW = q_block_words(QT, BS);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t blk = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; blk < nblocks; blk += stride) {
    uint32_t w[NW + 1];
    load_block_words<BB, NW>(packed + blk * BB, w);
    const float lo = half_bits_to_float(w[0] & 0xFFFFu);
    const float hi = half_bits_to_float(w[0] >> 16);
    const float step = __fdiv_rn(__fsub_rn(hi, lo), (float)D);
    float o[BS];
    bool bad = false;
#pragma unroll
    for (int j = 0; j < NC; j++) {
      const uint32_t v = get_code<C, NW>(w, j);
      if constexpr (QT == 35) {
        bad |= v > 120u;
        const uint32_t q1 = v / 11u;       // P:132 floor(q/11)
        const uint32_t q2 = v - 11u * q1;  // P:133 q mod 11
        o[2 * j] = __fmaf_rn((float)q1, step, lo);
        o[2 * j + 1] = __fmaf_rn((float)q2, step, lo);
      } else {
        o[j] = __fmaf_rn((float)v, step, lo);
      }
    }
    if (bad) report_status(dev_status, IF_ERR_DECODE);
    float4* dst = reinterpret_cast<float4*>(out + blk * BS);
#pragma unroll
    for (int i = 0; i < BS / 4; i++) dst[i] = make_float4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]);
  }
}

static int grid_for(int64_t items, int threads) {
  int64_t g = (items + threads - 1) / threads;
  const int64_t cap = 148 * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace ifb

using namespace ifb;

extern "C" if_status if_synth_fill(uint64_t seed, uint64_t tensor_id, float scale, float* out, int64_t n,
                                   int64_t offset, if_stream_t stream) {
  if (n < 0 || offset < 0) return set_error(IF_ERR_SHAPE, "if_synth_fill: n=%lld offset=%lld", (long long)n, (long long)offset);
  if (n == 0) return IF_OK;
  if (!out) return set_error(IF_ERR_ARG, "if_synth_fill: null out");
  const uint64_t base = seed ^ (tensor_id * 0x9E3779B97F4A7C15ull);
  synth_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(base, scale, out, n, offset);
  count_launch();
  return check_launch("if_synth_fill");
}

static if_status common_checks(const char* fn, if_scheme s, int64_t N, int64_t K, const void* a, const void* b) {
  if (!scheme_ok(s)) return set_error(IF_ERR_SCHEME, "%s: invalid scheme type=%d block=%d", fn, s.type, s.block);
  if (N < 0 || K < 0 || K % s.block) return set_error(IF_ERR_SHAPE, "%s: N=%lld K=%lld block=%d", fn, (long long)N, (long long)K, s.block);
  if (N * K > 0 && (!a || !b)) return set_error(IF_ERR_ARG, "%s: null pointer", fn);
  return IF_OK;
}

extern "C" if_status if_quantize(if_scheme s, const float* W, int64_t N, int64_t K, uint8_t* packed,
                                 int32_t* dev_status, if_stream_t stream) {
  if_status st = common_checks("if_quantize", s, N, K, W, packed);
  if (st) return st;
  if (N * K == 0) return IF_OK;
  if (reinterpret_cast<uintptr_t>(W) & 15u) return set_error(IF_ERR_ARG, "if_quantize: W must be 16-byte aligned");
  if ((q_block_bytes(s.type, s.block) % 4 == 0 && (reinterpret_cast<uintptr_t>(packed) & 3u)) ||
      (reinterpret_cast<uintptr_t>(packed) & 1u))
    return set_error(IF_ERR_ARG, "if_quantize: packed misaligned");
  const int64_t nblocks = N * (K / s.block);
  cudaStream_t cs = (cudaStream_t)stream;
  return dispatch_scheme(s, [&]<int QT, int BS>() -> if_status {
    quantize_kernel<QT, BS><<<grid_for(nblocks, 128), 128, 0, cs>>>(W, nblocks, packed, dev_status);
    count_launch();
    return check_launch("if_quantize");
  });
}

extern "C" if_status if_dequantize(if_scheme s, const uint8_t* packed, int64_t N, int64_t K, float* W_out,
                                   int32_t* dev_status, if_stream_t stream) {
  if_status st = common_checks("if_dequantize", s, N, K, packed, W_out);
  if (st) return st;
  if (N * K == 0) return IF_OK;
  if (reinterpret_cast<uintptr_t>(W_out) & 15u) return set_error(IF_ERR_ARG, "if_dequantize: W_out must be 16-byte aligned");
  if (reinterpret_cast<uintptr_t>(packed) & 1u) return set_error(IF_ERR_ARG, "if_dequantize: packed misaligned");
  const int64_t nblocks = N * (K / s.block);
  cudaStream_t cs = (cudaStream_t)stream;
  return dispatch_scheme(s, [&]<int QT, int BS>() -> if_status {
    dequantize_kernel<QT, BS><<<grid_for(nblocks, 128), 128, 0, cs>>>(packed, nblocks, W_out, dev_status);
    count_launch();
    return check_launch("if_dequantize");
  });
}
