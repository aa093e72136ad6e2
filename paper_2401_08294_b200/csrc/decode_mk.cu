// decode_mk.cu — persistent batch-1 decode engine for Q3H_B64 (the hot path).
//
// One CTA per SM, launched once per decode step.  The whole stack (or one
// standalone GEMV) is a sequence of phases; a phase is one fused-dequant GEMV
// (a4) whose input is produced by the previous phase, with the stack glue (a6)
// fused into the input staging and the output epilogue:
//
//   phase 4l+0  qkv  = W_qkv  rms(h)                   (x staged: h * 1/rms)
//   phase 4l+1  h   += W_o    vbcast(v)                (x staged: v of kv group)
//   phase 4l+2  gu   = W_gu   rms(h)
//   phase 4l+3  h   += W_down silu(g)*u
//
// Warp roles (B200-first):
//  * producer warp — one lane streams this CTA's row range of every phase, in
//    order, into a shared-memory ring with cp.async.bulk (the TMA engine),
//    completion tracked by mbarriers (full/empty per slot).  Weights never
//    depend on activations, so the producer runs ahead across phase and layer
//    boundaries and keeps HBM busy while consumers wait on a dependency.
//  * 8 consumer warps — wait until every CTA finished the previous phase (a
//    grid-wide counter, acquire/release at gpu scope), stage the transformed x
//    for the new phase in shared memory (identity (*) of simd.cuh), then decode
//    3.5-bit pair codes from the ring (2 SASS ops/weight) against x, R rows per
//    x load; partial sums are reduced with shuffles, combined across 32-block
//    chunks in a fixed order (deterministic), and written / residual-added.
// Rows of each phase are split evenly over the CTAs (contiguous ranges), so a
// CTA's share of a phase is one contiguous byte range of the packed tensor.
#include <stdlib.h>

#include <algorithm>
#include <utility>

#include "common.cuh"
#include "decode_mk.cuh"
#include "pipe.cuh"
#include "simd.cuh"
#include "mk_scheme.cuh"

namespace ifb {

#ifndef IFB_MK_NC
#define IFB_MK_NC 16
#endif
#ifndef IFB_MK_RMAX
#define IFB_MK_RMAX 4
#endif
constexpr int MK_NC = IFB_MK_NC;            // consumer warps
constexpr int MK_RMAX = IFB_MK_RMAX;        // rows per unit (x reuse)
constexpr int MK_THREADS = (MK_NC + 1) * 32;  // + producer warp
constexpr int MK_SLOT = 24 * 1024;          // ring slot bytes
constexpr int MK_MAXSLOT = 8;
#ifndef IFB_MK_INFLIGHT
#define IFB_MK_INFLIGHT 3
#endif
// slots the producer keeps in flight (issued, not landed).  Landed slots still
// fill the whole ring; bounding the bytes in flight bounds the queueing delay
// every other L2 access of this SM (the phase images, the tags) sees behind
// the weight stream (Little's law: ~3 slots cover the unloaded HBM latency).
constexpr int MK_INFLIGHT = IFB_MK_INFLIGHT;
constexpr int MK_CT = MK_NC * 32;           // consumer threads
constexpr int MK_MAXOWN = 256;              // residual rows owned by one CTA

struct Geo {
  int N, K, nb, nchunk, nbp, row_bytes, r0, r1, rps, R;
  int b0, coff, nchunk_all, full_row_bytes;  // K-segment: first block, chunk offset, all chunks, bytes of a whole row
};

// rows are split over the CTAs in contiguous balanced groups of `unit` rows
// (4 in stack mode: pairs of outputs for the transformed epilogue writes, and
// two (gate, up) row pairs = one act pair in the gate/up phase).  A phase whose K
// exceeds seg_nb blocks (70B down: K = 28672) runs in K-segments of seg_nb blocks
// (a multiple of 32: whole chunks), so the staged input in shared memory and the
// ring slots stay small; segment s covers blocks [s seg_nb, min(nb, (s+1) seg_nb)).
template <int BS = 64>
__device__ __forceinline__ int phase_nseg(int K, int seg_nb) {
  const int nb = BS == 64 ? K >> 6 : K >> 5;
  return seg_nb > 0 ? (nb + seg_nb - 1) / seg_nb : 1;
}
template <int BS = 64, int BB = 32, int RMAX = MK_RMAX>
__device__ __forceinline__ Geo phase_geo(int N, int K, int G, int cta, int unit, int seg_nb = 0, int sgi = 0) {
  Geo g;
  g.N = N;
  g.K = K;
  const int nb_all = BS == 64 ? K >> 6 : K >> 5;
  g.nchunk_all = (nb_all + 31) >> 5;
  g.full_row_bytes = nb_all * BB;
  g.b0 = seg_nb > 0 ? sgi * seg_nb : 0;
  g.nb = seg_nb > 0 ? min(seg_nb, nb_all - g.b0) : nb_all;
  g.coff = g.b0 >> 5;
  g.nchunk = (g.nb + 31) >> 5;
  g.nbp = g.nchunk << 5;
  g.row_bytes = g.nb * BB;
  const int units = N / unit;
  const int base = units / G, rem = units % G;
  g.r0 = (cta * base + min(cta, rem)) * unit;
  g.r1 = g.r0 + (base + (cta < rem ? 1 : 0)) * unit;
  int rps = MK_SLOT / g.row_bytes;
  if (RMAX >= 8 && rps >= 8) {
    g.R = 8;
    rps &= ~7;
  } else if (RMAX >= 4 && rps >= 4) {
    g.R = 4;
    rps &= ~3;
  } else if (rps >= 2) {
    g.R = 2;
    rps = 2;
  } else {
    g.R = 2;  // rows > 12 KB: one row per slot, the unit's second row is masked
    rps = 1;
  }
  g.rps = rps;
  return g;
}

__device__ __forceinline__ void phase_dims(const MkParams& P, int p, const uint8_t** W, int* N, int* K, int* kind) {
  if (P.mode == MK_MODE_GEMV) {
    *W = P.w[0][0];
    *N = P.gemv_N;
    *K = P.gemv_K;
    *kind = 4;
    return;
  }
  const int l = p >> 2, k = p & 3;
  *kind = k;
  *W = P.w[l][k];
  if (k == 0) {
    *N = P.nqkv;
    *K = P.d;
  } else if (k == 1) {
    *N = P.d;
    *K = P.nq;
  } else if (k == 2) {
    *N = 2 * P.lf;
    *K = P.d;
  } else {
    *N = P.d;
    *K = P.lf;
  }
}

// ---- consumer: R rows x one 32-block chunk ------------------------------------
// Sum over the 32 lanes of v[0..R) with a transposed butterfly; returns the sum
// of row (lane >> 3) on lanes 0, 8, 16, 24 (R = 4), row (lane >> 4) on lanes 0,
// 16 (R = 2), row 0 on lane 0 (R = 1).
template <int R>
__device__ __forceinline__ float warp_rows_sum(float (&v)[R]) {
  const int lane = threadIdx.x & 31;
  if constexpr (R == 8) {
    // 8 rows -> lanes 0,4,..,28 hold rows 0..7 (row = lane >> 2)
    const bool h16 = lane & 16;
    float a[4];
#pragma unroll
    for (int i = 0; i < 4; i++) {
      const float keep = h16 ? v[4 + i] : v[i], give = h16 ? v[i] : v[4 + i];
      a[i] = keep + __shfl_xor_sync(0xffffffffu, give, 16);
    }
    const bool h8 = lane & 8;
    float b0 = h8 ? a[2] : a[0], b1 = h8 ? a[3] : a[1];
    const float g0 = h8 ? a[0] : a[2], g1 = h8 ? a[1] : a[3];
    b0 += __shfl_xor_sync(0xffffffffu, g0, 8);
    b1 += __shfl_xor_sync(0xffffffffu, g1, 8);
    const bool h4 = lane & 4;
    float e = h4 ? b1 : b0;
    const float f = h4 ? b0 : b1;
    e += __shfl_xor_sync(0xffffffffu, f, 4);
    e += __shfl_xor_sync(0xffffffffu, e, 2);
    e += __shfl_xor_sync(0xffffffffu, e, 1);
    return e;
  } else if constexpr (R == 4) {
    const bool hi16 = lane & 16;
    float a = hi16 ? v[2] : v[0], b = hi16 ? v[3] : v[1];
    const float c = hi16 ? v[0] : v[2], d = hi16 ? v[1] : v[3];
    a += __shfl_xor_sync(0xffffffffu, c, 16);
    b += __shfl_xor_sync(0xffffffffu, d, 16);
    const bool hi8 = lane & 8;
    float e = hi8 ? b : a;
    const float f = hi8 ? a : b;
    e += __shfl_xor_sync(0xffffffffu, f, 8);
    e += __shfl_xor_sync(0xffffffffu, e, 4);
    e += __shfl_xor_sync(0xffffffffu, e, 2);
    e += __shfl_xor_sync(0xffffffffu, e, 1);
    return e;
  } else if constexpr (R == 2) {
    const bool hi16 = lane & 16;
    float a = hi16 ? v[1] : v[0];
    const float c = hi16 ? v[0] : v[1];
    a += __shfl_xor_sync(0xffffffffu, c, 16);
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    return a;
  } else {
    float a = v[0];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    return a;
  }
}

// One unit: R rows (R even) x one 32-block chunk, subnormal-form decode
// (simd.cuh).  XS = row stride of xs in float4 (compile time when XS > 0).
// FULL = every lane active and all R rows valid.
template <int R, int XS, bool FULL>
__device__ __forceinline__ void mk_unit(const unsigned char* slot_rows, int row_bytes, int nrows_valid, int c, int nb,
                                        int xs_rt, const float4* xs, const float2* bs, float* part_rows, int nchunk,
                                        const Q3HConst& kc) {
  static_assert(R % 2 == 0, "rows are paired in FFMA2 lanes");
  (void)kc;
  const int lane = threadIdx.x & 31;
  const int b = c * 32 + lane;
  const bool active = FULL || b < nb;
  const int xstride = XS > 0 ? XS : xs_rt;
  uint32_t wv[R][8];
#pragma unroll
  for (int i = 0; i < R; i++) {
    if (FULL || (active && i < nrows_valid)) {
      const uint4* a = reinterpret_cast<const uint4*>(slot_rows + i * row_bytes + b * 32);
      const uint4 lo = a[0], hi = a[1];
      wv[i][0] = lo.x; wv[i][1] = lo.y; wv[i][2] = lo.z; wv[i][3] = lo.w;
      wv[i][4] = hi.x; wv[i][5] = hi.y; wv[i][6] = hi.z; wv[i][7] = hi.w;
    } else {
#pragma unroll
      for (int k = 0; k < 8; k++) wv[i][k] = 0u;
    }
  }
  uint32_t vw[R][7];
#pragma unroll
  for (int i = 0; i < R; i++) {
    vw[i][0] = q3h_sview<0>(wv[i]); vw[i][1] = q3h_sview<1>(wv[i]); vw[i][2] = q3h_sview<2>(wv[i]);
    vw[i][3] = q3h_sview<3>(wv[i]); vw[i][4] = q3h_sview<4>(wv[i]); vw[i][5] = q3h_sview<5>(wv[i]);
    vw[i][6] = q3h_sview<6>(wv[i]);
  }
  u64 accc[R / 2], accq[R / 2];
#pragma unroll
  for (int i = 0; i < R / 2; i++) accc[i] = accq[i] = 0ull;
  const float4* xa = xs + b;
  float4 xn = xa[0];
#define IFB_MK_CODE(J, XC, XQ)                                                                  \
  {                                                                                             \
    constexpr uint32_t fm = q3h_floor_mult_bits(kQ3hSrc[J].pos);                                \
    const u64 fm2 = pack2(__uint_as_float(fm), __uint_as_float(fm));                            \
    const u64 xc2 = pack2(XC, XC), xq2 = pack2(XQ, XQ);                                         \
    _Pragma("unroll") for (int ip = 0; ip < R / 2; ip++) {                                      \
      const u64 cf = pack2(__uint_as_float(q3h_scode_bits<J>(wv[2 * ip], vw[2 * ip])),          \
                           __uint_as_float(q3h_scode_bits<J>(wv[2 * ip + 1], vw[2 * ip + 1]))); \
      const u64 qe = ffma2_rm(cf, fm2, 0ull);                                                   \
      accc[ip] = ffma2(cf, xc2, accc[ip]);                                                      \
      accq[ip] = ffma2(qe, xq2, accq[ip]);                                                      \
    }                                                                                           \
  }
#define IFB_MK_QUAD(JJ)                                                                         \
  {                                                                                             \
    const float4 xv = xn;                                                                       \
    if ((JJ) < 15) xn = xa[((JJ) + 1) * xstride]; /* prefetch the next x quad */                \
    IFB_MK_CODE(2 * (JJ), xv.x, xv.z)                                                           \
    IFB_MK_CODE(2 * (JJ) + 1, xv.y, xv.w)                                                       \
  }
  IFB_MK_QUAD(0) IFB_MK_QUAD(1) IFB_MK_QUAD(2) IFB_MK_QUAD(3) IFB_MK_QUAD(4) IFB_MK_QUAD(5)
  IFB_MK_QUAD(6) IFB_MK_QUAD(7) IFB_MK_QUAD(8) IFB_MK_QUAD(9) IFB_MK_QUAD(10) IFB_MK_QUAD(11)
  IFB_MK_QUAD(12) IFB_MK_QUAD(13) IFB_MK_QUAD(14) IFB_MK_QUAD(15)
#undef IFB_MK_QUAD
#undef IFB_MK_CODE
  const float sx = bs[b].x;
  float v[R];
#pragma unroll
  for (int ip = 0; ip < R / 2; ip++) {
    const float2 a = unpack2(accc[ip]), q = unpack2(accq[ip]);
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int i = 2 * ip + h;
      const float lo = half_bits_to_float(wv[i][0] & 0xFFFFu);
      const float hi = half_bits_to_float(wv[i][0] >> 16);
      // Eq. 2 with D = 10; 2^64 undoes the accumulator scale
      const float step = (hi - lo) * (0.1f * 18446744073709551616.0f);
      const float sq = h ? (a.y + q.y) : (a.x + q.x);
      const float r = fmaf(step, sq, lo * sx);
      v[i] = active ? r : 0.f;
    }
  }
  const float sum = warp_rows_sum<R>(v);
  constexpr int SH = R == 8 ? 2 : (R == 4 ? 3 : (R == 2 ? 4 : 5));
  const int row = lane >> SH;
  if ((lane & ((1 << SH) - 1)) == 0 && (FULL || row < nrows_valid)) part_rows[row * nchunk + c] = sum;
}

template <int R, int XS>
__device__ __forceinline__ void mk_unit_dispatch(const unsigned char* slot_rows, int row_bytes, int nrows_valid, int c,
                                                 int nb, int xs_rt, const float4* xs, const float2* bs,
                                                 float* part_rows, int nchunk, const Q3HConst& kc) {
  if (nrows_valid >= R && (c + 1) * 32 <= nb)
    mk_unit<R, XS, true>(slot_rows, row_bytes, nrows_valid, c, nb, xs_rt, xs, bs, part_rows, nchunk, kc);
  else
    mk_unit<R, XS, false>(slot_rows, row_bytes, nrows_valid, c, nb, xs_rt, xs, bs, part_rows, nchunk, kc);
}

template <int W, int BS, int NWP, int NV, int... V>
__device__ __forceinline__ void gk_views(std::integer_sequence<int, V...>, const uint32_t (&w)[NWP], uint32_t (&vw)[NV]) {
  ((vw[V] = gk_view<W, BS, V>(w)), ...);
}
// quad J of a k-bit unit: codes 4J..4J+3 of R rows against the staged X of quad J
template <int W, int BS, int R, int NWP, int NV, int J, int... I>
__device__ __forceinline__ void gk_quad(std::integer_sequence<int, I...>, const float4& xv, const uint32_t (&wv)[R][NWP],
                                        const uint32_t (&vw)[R][NV], u64 (&acc)[R / 2][2]) {
  const float xc[4] = {xv.x, xv.y, xv.z, xv.w};
  (
      [&] {
        constexpr int K = 4 * J + I;
        const u64 x2 = pack2(xc[I], xc[I]);
#pragma unroll
        for (int ip = 0; ip < R / 2; ip++) {
          const u64 cf = pack2(__uint_as_float(gk_code_bits<W, BS, K>(wv[2 * ip], vw[2 * ip])),
                               __uint_as_float(gk_code_bits<W, BS, K>(wv[2 * ip + 1], vw[2 * ip + 1])));
          acc[ip][K & 1] = ffma2(cf, x2, acc[ip][K & 1]);
        }
      }(),
      ...);
}
template <int W, int BS, int R, int NWP, int NV, int... J>
__device__ __forceinline__ void gk_quads(std::integer_sequence<int, J...>, const float4* xa, int xstride, float4& xn,
                                         const uint32_t (&wv)[R][NWP], const uint32_t (&vw)[R][NV],
                                         u64 (&acc)[R / 2][2]) {
  constexpr int NQ = sizeof...(J);
  (
      [&] {
        const float4 xv = xn;
        if constexpr (J + 1 < NQ) xn = xa[(J + 1) * xstride];  // prefetch the next quad
        gk_quad<W, BS, R, NWP, NV, J>(std::make_integer_sequence<int, 4>{}, xv, wv, vw, acc);
      }(),
      ...);
}

// ---- k-bit schemes (mk_scheme.cuh): one unit = R rows x one 32-block chunk ----------
// Lane = block b of the chunk; X_k = x_k 2^(85 - s_k) staged as quads of 4 codes.
template <int W, int BS, int R, int XS, bool FULL>
__device__ __forceinline__ void gk_unit(const unsigned char* slot_rows, int row_bytes, int nrows_valid, int c, int nb,
                                        int xs_rt, const float4* xs, const float2* bs, float* part_rows, int nchunk) {
  using S = GkScheme<W, BS>;
  static_assert(R % 2 == 0, "rows are paired in FFMA2 lanes");
  constexpr int NW = S::NW, NV = S::NV > 0 ? S::NV : 1;
  const int lane = threadIdx.x & 31;
  const int b = c * 32 + lane;
  const bool active = FULL || b < nb;
  const int xstride = XS > 0 ? XS : xs_rt;
  uint32_t wv[R][NW + 1];
#pragma unroll
  for (int i = 0; i < R; i++) {
    const bool ok = FULL || (active && i < nrows_valid);
    const unsigned char* a = slot_rows + i * row_bytes + b * S::BB;
    if constexpr (S::BB % 16 == 0) {
#pragma unroll
      for (int q = 0; q < NW / 4; q++) {
        uint4 v = ok ? reinterpret_cast<const uint4*>(a)[q] : make_uint4(0u, 0u, 0u, 0u);
        wv[i][4 * q] = v.x; wv[i][4 * q + 1] = v.y; wv[i][4 * q + 2] = v.z; wv[i][4 * q + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int q = 0; q < NW; q++) wv[i][q] = ok ? reinterpret_cast<const uint32_t*>(a)[q] : 0u;
    }
    wv[i][NW] = 0u;
  }
  uint32_t vw[R][NV];
#pragma unroll
  for (int i = 0; i < R; i++) gk_views<W, BS>(std::make_integer_sequence<int, S::NV>{}, wv[i], vw[i]);
  u64 acc[R / 2][2];
#pragma unroll
  for (int i = 0; i < R / 2; i++) acc[i][0] = acc[i][1] = 0ull;
  const float4* xa = xs + b;
  float4 xn = xa[0];
  gk_quads<W, BS, R, NW + 1, NV>(std::make_integer_sequence<int, S::NQ>{}, xa, xstride, xn, wv, vw, acc);
  const float sx = bs[b].x;
  float v[R];
#pragma unroll
  for (int ip = 0; ip < R / 2; ip++) {
    const float2 a0 = unpack2(acc[ip][0]), a1 = unpack2(acc[ip][1]);
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int i = 2 * ip + h;
      const float lo = half_bits_to_float(wv[i][0] & 0xFFFFu);
      const float hi = half_bits_to_float(wv[i][0] >> 16);
      // Eq. 2: step = (hi - lo) / D; 2^64 undoes the accumulator scale
      const float step = (hi - lo) * (18446744073709551616.0f / (float)S::D);
      const float sq = h ? (a0.y + a1.y) : (a0.x + a1.x);
      v[i] = active ? fmaf(step, sq, lo * sx) : 0.f;
    }
  }
  const float sum = warp_rows_sum<R>(v);
  constexpr int SH = R == 8 ? 2 : (R == 4 ? 3 : (R == 2 ? 4 : 5));
  const int row = lane >> SH;
  if ((lane & ((1 << SH) - 1)) == 0 && (FULL || row < nrows_valid)) part_rows[row * nchunk + c] = sum;
}

// scheme-dispatched pieces of the engine: QT = 35 is the paper's 3.5-bit pair code
// (the subnormal-form pair decode above), QT = k a k-bit scheme (mk_scheme.cuh)
template <int QT, int BS, int R, int XS>
__device__ __forceinline__ void sk_unit_dispatch(const unsigned char* slot_rows, int row_bytes, int nrows_valid, int c,
                                                 int nb, int xs_rt, const float4* xs, const float2* bs,
                                                 float* part_rows, int nchunk, const Q3HConst& kc) {
  if constexpr (QT == 35) {
    mk_unit_dispatch<R, XS>(slot_rows, row_bytes, nrows_valid, c, nb, xs_rt, xs, bs, part_rows, nchunk, kc);
  } else {
    constexpr int RR = R > GkScheme<QT, BS>::RMAX ? GkScheme<QT, BS>::RMAX : R;
    if (nrows_valid >= RR && (c + 1) * 32 <= nb)
      gk_unit<QT, BS, RR, XS, true>(slot_rows, row_bytes, nrows_valid, c, nb, xs_rt, xs, bs, part_rows, nchunk);
    else
      gk_unit<QT, BS, RR, XS, false>(slot_rows, row_bytes, nrows_valid, c, nb, xs_rt, xs, bs, part_rows, nchunk);
  }
}

// code bit position s_j of pair j (simd.cuh kQ3hSrc), for the per-pair x scaling;
// copied to shared memory at kernel start (lanes index it with different j)
__device__ const int kQ3hPosTab[32] = {0, 7, 14, 0, 7, 3, 10, 17, 0, 7, 6, 13, 0, 7, 2, 9,
                                       16, 0, 7, 5, 12, 0, 7, 1, 8, 15, 0, 7, 4, 11, 0, 7};
constexpr int MK_MAXQ = 8;  // staged quads held in registers per consumer thread

// Stage one quad of x: weights 4q..4q+3 = pairs 2JJ, 2JJ+1 of block b = q / 16,
// JJ = q % 16:
//   xs[JJ * xstride + b] = {X_c(2JJ), X_c(2JJ+1), X_q(2JJ), X_q(2JJ+1)}
//   X_c(j) = x_o(j) * 2^(85 - s_j),   X_q(j) = (x_e(j) - 11 x_o(j)) * 2^85
// (subnormal-form decode, simd.cuh) and bs[b].x = sum of the block's 64 x.
// xstride = 1 (mod 8) makes the transposed stores conflict-free; a block's 16
// quads sit in one half-warp (all 32 lanes must call this together).
__device__ __forceinline__ void stage_quad(int q, float4 v, int xstride, float4* xs, float2* bs, const int* pos) {
  const int b = q >> 4, jj = q & 15;
  const float s85 = 38685626227668133590597632.0f;  // 2^85
  const float c0 = __uint_as_float((uint32_t)(127 + 85 - pos[2 * jj]) << 23);
  const float c1 = __uint_as_float((uint32_t)(127 + 85 - pos[2 * jj + 1]) << 23);
  // pairs (v.x, v.y) and (v.z, v.w): x_e = .x/.z, x_o = .y/.w
  xs[jj * xstride + b] = make_float4(v.y * c0, v.w * c1, fmaf(-11.0f, v.y, v.x) * s85, fmaf(-11.0f, v.w, v.z) * s85);
  float sx = (v.x + v.y) + (v.z + v.w);
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) sx += __shfl_xor_sync(0xffffffffu, sx, o);
  if (jj == 0) bs[b] = make_float2(sx, 0.f);
}

// 1 / sqrt(mean(h^2) + 1e-5) from every consumer thread's partial sum of squares
__device__ __forceinline__ float mk_rms_inv(float ss, float* red, int K, int cw, int lane) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if (lane == 0) red[cw] = ss;
  named_bar_sync(1, MK_CT);
  float tot = 0.f;
#pragma unroll
  for (int w = 0; w < MK_NC; w++) tot += red[w];
  return 1.0f / sqrtf(tot / (float)K + 1e-5f);
}

// ---- scheme-dispatched staging (sk_*): QT = 35 the pair transform above, else X_k ----
template <int QT, int BS>
struct SkTraits {  // staged quads per block, block bytes, code positions kept in shared memory
  static constexpr int NQ = QT == 35 ? 16 : BS / 4;
  static constexpr int BB = QT == 35 ? 32 : GkScheme<QT, BS>::BB;
  static constexpr int NPOS = QT == 35 ? 32 : BS;
  static constexpr int RMAX = QT == 35 ? MK_RMAX : GkScheme<QT, BS>::RMAX;
};

// k-bit stage: quad q = weights 4q..4q+3 of the input -> X_k = x_k 2^(85 - s_k)
template <int QT, int BS>
__device__ __forceinline__ void sk_stage_quad(int q, float4 v, int xstride, float4* xs, float2* bs, const int* pos) {
  if constexpr (QT == 35) {
    stage_quad(q, v, xstride, xs, bs, pos);
  } else {
    constexpr int NQ = BS / 4;
    const int b = q / NQ, jj = q % NQ;
    const int* p = pos + 4 * jj;
    xs[jj * xstride + b] = make_float4(v.x * __uint_as_float((uint32_t)(127 + 85 - p[0]) << 23),
                                       v.y * __uint_as_float((uint32_t)(127 + 85 - p[1]) << 23),
                                       v.z * __uint_as_float((uint32_t)(127 + 85 - p[2]) << 23),
                                       v.w * __uint_as_float((uint32_t)(127 + 85 - p[3]) << 23));
    float sx = (v.x + v.y) + (v.z + v.w);
#pragma unroll
    for (int o = NQ / 2; o > 0; o >>= 1) sx += __shfl_xor_sync(0xffffffffu, sx, o);
    if (jj == 0) bs[b] = make_float2(sx, 0.f);
  }
}

// sum of the four x values a staged quad jj encodes (image staging: the block sums)
template <int QT, int BS>
__device__ __forceinline__ float sk_quad_sum(float4 w, int jj, const int* pos) {
  if constexpr (QT == 35) {
    const float c0 = __uint_as_float((uint32_t)(127 - 85 + pos[2 * jj]) << 23);  // 2^(s - 85)
    const float c1 = __uint_as_float((uint32_t)(127 - 85 + pos[2 * jj + 1]) << 23);
    return (w.z + w.w) * 2.5849394142282115e-26f + 12.0f * (w.x * c0 + w.y * c1);
  } else {
    const int* p = pos + 4 * jj;
    return (w.x * __uint_as_float((uint32_t)(127 - 85 + p[0]) << 23) + w.y * __uint_as_float((uint32_t)(127 - 85 + p[1]) << 23)) +
           (w.z * __uint_as_float((uint32_t)(127 - 85 + p[2]) << 23) + w.w * __uint_as_float((uint32_t)(127 - 85 + p[3]) << 23));
  }
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// ---- phase images: readiness carried by the data itself ------------------------
// A phase's input vector is written by the previous phase's epilogues, each CTA
// its own rows, straight into a global "image" in the transformed quad layout of
// stage_quad.  Every stored float carries the image version's parity in its
// mantissa LSB (stripped by the reader: values do not depend on it), and the
// stores are single-copy-atomic 32-bit words, so a reader that sees the
// expected parity in a word sees that word's final value.  The writer needs no
// fence: after its epilogue it bumps a relaxed per-phase counter; a reader waits
// for the counter (every CTA past the phase = every CTA done reading the
// previous version: 1-bit parity cannot alias), bulk-copies the image and
// re-reads (ld.relaxed.gpu, L1 bypassed) the rare word whose store had not
// landed yet.
__device__ __forceinline__ float4 ld_relaxed_f4(const float4* p) {
  float4 v;
  asm volatile("ld.relaxed.gpu.global.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u32(void* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// system-scope relaxed accesses for the TP exchange regions (peer GPU memory over NVLink)
__device__ __forceinline__ uint32_t ld_relaxed_sys_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys_u32(void* p, uint32_t v) {
  asm volatile("st.relaxed.sys.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// value with its mantissa LSB replaced by the image parity
__device__ __forceinline__ uint32_t tagp(float v, uint32_t par) { return (__float_as_uint(v) & ~1u) | par; }
__device__ __forceinline__ bool par4_ok(float4 v, uint32_t par) {
  return (((__float_as_uint(v.x) ^ par) | (__float_as_uint(v.y) ^ par) | (__float_as_uint(v.z) ^ par) |
           (__float_as_uint(v.w) ^ par)) & 1u) == 0u;
}
// a wait that never ends is a bug (or a workspace that was not zero-filled):
// trap after ~2 s instead of hanging the GPU
struct SpinGuard {
  uint32_t n = 0;
  unsigned long long t0 = 0;
  __device__ __forceinline__ void tick() {
    if ((++n & 255u) == 0u) {
      const unsigned long long t = gtimer();
      if (n == 256u) t0 = t;
      else if (t - t0 > 2000000000ull) __trap();
    }
  }
};

// Write the transformed pair (x_e, x_o) of element k (k even) of a phase input
// into a global image with the shared-memory layout of stage_quad, tagged with
// the image parity.
__device__ __forceinline__ void put_pair(float4* xsg, int xstride, const int* pos, int k, float xe, float xo,
                                         uint32_t par) {
  const int b = k >> 6, j = (k >> 1) & 31, jj = j >> 1, comp = j & 1;
  float* f = reinterpret_cast<float*>(xsg + jj * xstride + b);
  const float cj = __uint_as_float((uint32_t)(127 + 85 - pos[j]) << 23);  // 2^(85 - s_j)
  st_relaxed_u32(f + comp, tagp(xo * cj, par));
  st_relaxed_u32(f + 2 + comp, tagp(fmaf(-11.0f, xo, xe) * 38685626227668133590597632.0f, par));  // * 2^85
}

template <int QT, int BS>
__device__ __forceinline__ void sk_put_pair(float4* xsg, int xstride, const int* pos, int k, float xe, float xo,
                                            uint32_t par) {
  if constexpr (QT == 35) {
    put_pair(xsg, xstride, pos, k, xe, xo, par);
  } else {
    // elements k, k+1 (k even) -> components k % 4, k % 4 + 1 of quad (k % BS) / 4 of block k / BS
    const int b = k / BS, kk = k % BS, jj = kk >> 2, comp = kk & 3;
    float* f = reinterpret_cast<float*>(xsg + jj * xstride + b) + comp;
    st_relaxed_u32(f, tagp(xe * __uint_as_float((uint32_t)(127 + 85 - pos[kk]) << 23), par));
    st_relaxed_u32(f + 1, tagp(xo * __uint_as_float((uint32_t)(127 + 85 - pos[kk + 1]) << 23), par));
  }
}

template <int XS, bool SEG, bool TP = false, int QT = 35, int BS = 64, bool PL = false>
__global__ void __launch_bounds__(MK_THREADS, 1) decode_mk_kernel(const __grid_constant__ MkParams P) {
  using SK = SkTraits<QT, BS>;
  const int xstride = XS > 0 ? XS : P.xstride;  // staged input in shared memory
  const int xg = SEG ? P.xg : xstride;            // global phase images (whole K; = xstride unless segmented)
  extern __shared__ __align__(1024) unsigned char smem[];
  const int G = gridDim.x, cta = blockIdx.x;
  const int nslot = P.nslot;
  unsigned char* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)nslot * MK_SLOT);
  uint64_t* empty = full + MK_MAXSLOT;
  float* red = reinterpret_cast<float*>(empty + MK_MAXSLOT);  // [MK_NC] + scalars
  float4* xs = reinterpret_cast<float4*>(smem + (size_t)nslot * MK_SLOT + 2 * MK_MAXSLOT * 8 + 128);
  float2* bs = reinterpret_cast<float2*>(xs + SK::NQ * xstride);
  float* h_own = reinterpret_cast<float*>(bs + P.nbp_max);    // [MK_MAXOWN] this CTA's residual rows
  int* pos = reinterpret_cast<int*>(h_own + MK_MAXOWN);       // [32] code positions
  float* ssq_s = reinterpret_cast<float*>(pos + SK::NPOS);          // [MK_MAXG] sum h^2 partials
  float* part = ssq_s + MK_MAXG;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nslot; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MK_NC);  // every consumer warp arrives once per fill
    }
    fence_mbar_init();
  }
  if constexpr (QT == 35) {
    if (threadIdx.x < 32) pos[threadIdx.x] = kQ3hPosTab[threadIdx.x];
  } else {
    [&]<int... K>(std::integer_sequence<int, K...>) {
      ((threadIdx.x == K ? (void)(pos[K] = GkSrc<QT, BS, K>::pos) : (void)0), ...);
    }(std::make_integer_sequence<int, BS>{});
  }
  __syncthreads();
  if constexpr (PL) pdl_trigger();
  const bool stack = P.mode == MK_MODE_STACK;
  const int nphase = stack ? 4 * P.layers : 1;
  const int pb = PL ? P.p_begin : 0, pe = PL ? P.p_end : nphase;  // this launch's phases
  const int unit = stack ? 4 : 1;

  if (warp == 0) {
    // ============================ producer ============================
#ifdef IFB_MK_NOWAIT
    if (false) {
#else
    if (lane == 0) {
#endif
      const uint64_t pol = policy_evict_first();
      uint32_t slot = 0, round = 0, seq = 0;
      for (int p = pb; p < pe; p++) {
        const uint8_t* W;
        int N, K, kind;
        phase_dims(P, p, &W, &N, &K, &kind);
        const int nseg = SEG ? phase_nseg<BS>(K, P.seg_nb) : 1;
        for (int sgi = 0; sgi < nseg; sgi++) {
          const Geo g = phase_geo<BS, SK::BB, SK::RMAX>(N, K, G, cta, unit, SEG && nseg > 1 ? P.seg_nb : 0, sgi);
          for (int r = g.r0; r < g.r1; r += g.rps) {
            const int n = min(g.rps, g.r1 - r);
            const uint32_t bytes = (uint32_t)n * g.row_bytes;
            if (MK_INFLIGHT < nslot && seq >= (uint32_t)MK_INFLIGHT) {
              const uint32_t q = seq - MK_INFLIGHT;  // the copy MK_INFLIGHT issues ago must have landed
              mbar_wait_sleep(&full[q % (uint32_t)nslot], (q / (uint32_t)nslot) & 1);
            }
            seq++;
            mbar_wait_sleep(&empty[slot], (round & 1) ^ 1);
            mbar_arrive_expect_tx(&full[slot], bytes);
            if (nseg == 1) {  // contiguous rows: one copy
              bulk_g2s(ring + (size_t)slot * MK_SLOT, W + (size_t)r * g.row_bytes, bytes, &full[slot], pol);
            } else {  // a K-segment of each row: one copy per row
              for (int i = 0; i < n; i++)
                bulk_g2s(ring + (size_t)slot * MK_SLOT + (size_t)i * g.row_bytes,
                         W + (size_t)(r + i) * g.full_row_bytes + (size_t)g.b0 * SK::BB, (uint32_t)g.row_bytes,
                         &full[slot], pol);
            }
            if (++slot == (uint32_t)nslot) {
              slot = 0;
              round++;
            }
          }
        }
      }
    }
    return;
  }

  // ============================ consumers ============================
  if constexpr (PL) pdl_wait();  // the predecessor (attention) wrote this launch's inputs
  const int ct = threadIdx.x - 32;
  const int cw = warp - 1;
  const Q3HConst kc = q3h_const();
  uint32_t slot = 0, round = 0;  // ring position (same sequence as the producer)
  // image versions of this launch (decode_mk.cuh): ctx/act are written once per
  // layer, h (and the sum-h^2 partials) twice; version 0 = the zero-filled workspace
  const uint32_t ep = stack ? ld_relaxed_u32(P.epoch) : 0u;
  const uint32_t L2 = 2u * (uint32_t)P.layers;
  if (stack) {
    // residual rows of this CTA (the o/down row split) from the stage input
    const Geo go = phase_geo<BS, SK::BB, SK::RMAX>(P.d, P.nq, G, cta, unit);
    for (int i = ct; i < go.r1 - go.r0; i += MK_CT) h_own[i] = P.h[go.r0 + i];
  }
  for (int p = pb; p < pe; p++) {
    if constexpr (SEG) {
    const uint8_t* W;
    int N, K, kind;
    phase_dims(P, p, &W, &N, &K, &kind);
    const int nseg = SEG ? phase_nseg<BS>(K, P.seg_nb) : 1;
    (void)W;
    unsigned long long* dbg = P.dbg ? P.dbg + ((size_t)cta * nphase + p) * 16 : nullptr;
    if (dbg && ct == 0) { dbg[0] = gtimer(); dbg[8] = clock64(); }
    // Phase input.  Producers (the previous phase's epilogues) already wrote it in
    // the transformed quad layout into a global xs image: one dependency wait, then
    // 16 bulk copies (one per quad row JJ) + the sum-h^2 partials for RMSNorm.
    // The first phase (plain h) and the standalone GEMV stage from global memory.
    const bool from_image = stack && p > pb;
    const bool rms = kind == 0 || kind == 2;
    const uint32_t l = (uint32_t)(p >> 2);
    float out_scale = 1.f;  // RMSNorm folded into the output: W (s h) = s (W h)
    const float4* img = nullptr;
    uint32_t par = 0;
    if (from_image) {
      // input image of this phase and the version its writers tag it with
      uint32_t ver;
      if (kind == 1) {
        img = P.xs_ctx, ver = ep * (uint32_t)P.layers + l + 1u;
      } else if (kind == 3) {
        img = P.xs_act, ver = ep * (uint32_t)P.layers + l + 1u;
      } else {
        img = P.xs_h, ver = ep * L2 + 2u * l + (kind == 2 ? 1u : 0u);  // kind 0: down of layer l-1
      }
      par = ver & 1u;
      // 1. one thread waits until every CTA has finished the previous phase (a
      //    relaxed counter: no fence on either side -- the data carries its own
      //    readiness); IFB_MK_POLL: no counter, every thread polls its own words
#ifndef IFB_MK_POLL
      if (ct == 0) {
        SpinGuard sg;
        const uint32_t target = (ep + 1u) * (uint32_t)G - (uint32_t)P.early;
        // wrap-safe: the difference is taken in uint32_t (defined modulo 2^32), then read as signed
        while ((int32_t)(ld_relaxed_u32(reinterpret_cast<const uint32_t*>(P.done + p - 1)) - target) < 0) {
          __nanosleep(20);
          sg.tick();
        }
      }
      named_bar_sync(1, MK_CT);
#endif
      if (dbg && ct == 0) { dbg[1] = gtimer(); dbg[9] = clock64(); }
      // 2. the sum-h^2 partials, read straight from L2 (ld.relaxed.gpu bypasses L1),
      //    parity-checked like the image; fixed order: deterministic
      if (rms && cw == MK_NC - 1) {
        // all loads in flight at once (G <= MK_MAXG = 5 x 32), then check / re-read
        constexpr int NS = (MK_MAXG + 31) / 32;
        uint32_t sv[NS];
#pragma unroll
        for (int i = 0; i < NS; i++)
          sv[i] = lane + 32 * i < G ? ld_relaxed_u32(reinterpret_cast<const uint32_t*>(P.ssq) + lane + 32 * i) : par;
        float t = 0.f;
#pragma unroll
        for (int i = 0; i < NS; i++) {
          const int c = lane + 32 * i;
          uint32_t v = sv[i];
          if (c >= G) continue;
          if ((v ^ par) & 1u) {
            SpinGuard sg;
            do {
              __nanosleep(32);
              sg.tick();
              v = ld_relaxed_u32(reinterpret_cast<const uint32_t*>(P.ssq) + c);
            } while ((v ^ par) & 1u);
          }
          t += __uint_as_float(v & ~1u);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0) red[16] = t;
      }
      if (dbg && ct == 0) { dbg[6] = gtimer(); dbg[14] = clock64(); }
    }
    float plain_inv = 1.f;
    for (int sgi = 0; sgi < nseg; sgi++) {
    const Geo g = phase_geo<BS, SK::BB, SK::RMAX>(N, K, G, cta, unit, SEG && nseg > 1 ? P.seg_nb : 0, sgi);
    if (sgi > 0) named_bar_sync(1, MK_CT);  // every warp is done with the previous segment's xs
    if (from_image) {
      // 3. four threads per block b, four quads each: load the image words straight
      //    from L2 into registers (all loads of a thread in flight at once), check
      //    every word's parity (re-read the late ones), strip it, stage the quads in
      //    shared memory and form the block sum of x (x_e + x_o = xe' + 12 x_o in
      //    transformed terms)
      constexpr int TPB = SK::NQ / 4, TPB_LOG = TPB == 4 ? 2 : 1;  // threads per block, 4 quads each
      for (int t0 = cw * 32; t0 < TPB * g.nbp; t0 += 2 * MK_CT) {
        float4 v[2][4];
#pragma unroll
        for (int u = 0; u < 2; u++) {
          const int t = t0 + u * MK_CT + lane, b = t >> TPB_LOG, j4 = t & (TPB - 1);
#pragma unroll
          for (int i = 0; i < 4; i++)
            v[u][i] = b < g.nb ? ld_relaxed_f4(img + (4 * j4 + i) * xg + g.b0 + b) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < 2; u++) {
          if (t0 + u * MK_CT >= TPB * g.nbp) break;  // warp-uniform
          const int t = t0 + u * MK_CT + lane, b = t >> TPB_LOG, j4 = t & (TPB - 1);
          float sx = 0.f;
          if (b < g.nb) {
#pragma unroll
            for (int i = 0; i < 4; i++) {
              const int jj = 4 * j4 + i;
              float4 q = v[u][i];
              if (!par4_ok(q, par)) {
                SpinGuard sg;
                do {
                  if (dbg) atomicAdd(reinterpret_cast<unsigned long long*>(dbg + 7), 1ull);
                  __nanosleep(32);
                  sg.tick();
                  q = ld_relaxed_f4(img + jj * xg + g.b0 + b);
                } while (!par4_ok(q, par));
              }
              const float4 w = make_float4(__uint_as_float(__float_as_uint(q.x) & ~1u), __uint_as_float(__float_as_uint(q.y) & ~1u),
                                           __uint_as_float(__float_as_uint(q.z) & ~1u), __uint_as_float(__float_as_uint(q.w) & ~1u));
              xs[jj * xstride + b] = w;
              sx += sk_quad_sum<QT, BS>(w, jj, pos);
            }
          }
          sx += __shfl_xor_sync(0xffffffffu, sx, 1);
          if constexpr (TPB > 2) sx += __shfl_xor_sync(0xffffffffu, sx, 2);
          if (j4 == 0 && b < g.nbp) bs[b] = make_float2(sx, 0.f);
        }
      }
      if (dbg && ct == 0) { dbg[2] = gtimer(); dbg[10] = clock64(); }
      named_bar_sync(1, MK_CT);
      if (rms && sgi == 0) out_scale = 1.0f / sqrtf(red[16] / (float)K + 1e-5f);
    } else {
      // plain input (stage input h, or the GEMV's x) read straight from global memory
      // (coalesced 128-bit loads, L2 hits after the first CTA) and staged as
      // transformed quads; no shared-memory copy of the raw vector, so the largest
      // shapes (70B: K up to 28672) fit.  RMSNorm needs the global sum of squares
      // first: quads stay in registers when they fit, else they are re-read.
      const float4* src4 = reinterpret_cast<const float4*>(stack ? P.h : P.x_in) + (size_t)g.b0 * (BS / 4);
      const int nq = K >> 2, nqs = g.nb * SK::NQ, nqp = g.nbp * SK::NQ;
      if (rms && nseg == 1 && nqp <= MK_MAXQ * MK_CT) {
        float4 v[MK_MAXQ];
        float ss = 0.f;
#pragma unroll
        for (int i = 0; i < MK_MAXQ; i++) {
          const int q = ct + i * MK_CT;
          v[i] = q < nq ? src4[q] : make_float4(0.f, 0.f, 0.f, 0.f);
          ss = fmaf(v[i].x, v[i].x, fmaf(v[i].y, v[i].y, fmaf(v[i].z, v[i].z, fmaf(v[i].w, v[i].w, ss))));
        }
        plain_inv = mk_rms_inv(ss, red, K, cw, lane);
#pragma unroll
        for (int i = 0; i < MK_MAXQ; i++)
          if (i * MK_CT + (ct & ~31) < nqp) {  // per-warp (nqp is a multiple of 32)
            const float4 a = v[i];
            const float inv = plain_inv;
            sk_stage_quad<QT, BS>(ct + i * MK_CT, make_float4(a.x * inv, a.y * inv, a.z * inv, a.w * inv), xstride, xs, bs, pos);
          }
      } else {
        if (rms && sgi == 0) {
          const float4* all4 = reinterpret_cast<const float4*>(stack ? P.h : P.x_in);
          float ss = 0.f;
          for (int q = ct; q < nq; q += MK_CT) {
            const float4 a = all4[q];
            ss = fmaf(a.x, a.x, fmaf(a.y, a.y, fmaf(a.z, a.z, fmaf(a.w, a.w, ss))));
          }
          plain_inv = mk_rms_inv(ss, red, K, cw, lane);
        }
        const float inv = plain_inv;
        for (int q = ct; q < nqp; q += MK_CT) {
          float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
          if (q < nqs) a = src4[q];
          sk_stage_quad<QT, BS>(q, make_float4(a.x * inv, a.y * inv, a.z * inv, a.w * inv), xstride, xs, bs, pos);
        }
      }
      if (dbg && ct == 0) { dbg[2] = gtimer(); dbg[10] = clock64(); }
      named_bar_sync(1, MK_CT);
    }
    if (dbg && ct == 0) { dbg[3] = gtimer(); dbg[11] = clock64(); }
    // ---- 3. stream this CTA's rows from the ring.  Every consumer warp visits
    //         every slot (wait full -> its units -> arrive empty, count NC);
    //         the units (R rows x one chunk) of consecutive slots are dealt
    //         round-robin over the warps: global unit t = sl*U + u -> warp t % NC.
    {
      const int nrows = g.r1 - g.r0;
      const int nslots = (nrows + g.rps - 1) / g.rps;
      const int gps = max(1, g.rps / g.R);         // row groups per full slot (rps = 1 < R: one masked group)
      const int U = gps * g.nchunk;                // units per slot
      const int inv_nc = (65536 + g.nchunk - 1) / g.nchunk;
      int u0 = cw;                                 // first unit of this warp in slot sl
#ifdef IFB_MK_PROF
      // instrumentation: ring slots of this phase already landed at stream start, and
      // clocks warp 0 spends waiting for slots (-> dbg[15] = wait << 8 | occupancy)
      unsigned long long pw = 0;
      uint32_t occ = 0;
      if (dbg && ct == 0) {
        uint32_t s2 = slot, r2 = round;
        for (int i = 0; i < nslots && i < nslot; i++) {
          uint32_t ok;
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                       : "=r"(ok) : "r"(smem_u32(&full[s2])), "r"(r2 & 1) : "memory");
          if (!ok) break;
          occ++;
          if (++s2 == (uint32_t)nslot) { s2 = 0; r2++; }
        }
      }
#endif
      for (int sl = 0; sl < nslots; sl++) {
#ifdef IFB_MK_PROF
        const unsigned long long pw0 = clock64();
#endif
#ifndef IFB_MK_NOWAIT
        mbar_wait_sleep(&full[slot], round & 1);
#endif
#ifdef IFB_MK_PROF
        pw += clock64() - pw0;
#endif
        const int n = min(g.rps, nrows - sl * g.rps);
        const unsigned char* sbase = ring + (size_t)slot * MK_SLOT;
        int u = u0;
        for (; u < U; u += MK_NC) {
          const int grp = (u * inv_nc) >> 16, c = u - grp * g.nchunk;
          const int i0 = grp * g.R;
#ifdef IFB_MK_NOCOMPUTE
          if (false) {
#else
          if (i0 < n) {
#endif
            float* pr = part + (size_t)(sl * g.rps + i0) * g.nchunk_all + g.coff;
            const unsigned char* ua = sbase + (size_t)i0 * g.row_bytes;
            if (MK_RMAX >= 8 && g.R == 8)
              sk_unit_dispatch<QT, BS, MK_RMAX >= 8 ? 8 : 4, XS>(ua, g.row_bytes, n - i0, c, g.nb, xstride, xs, bs, pr, g.nchunk_all, kc);
            else if (g.R == 4)
              sk_unit_dispatch<QT, BS, 4, XS>(ua, g.row_bytes, n - i0, c, g.nb, xstride, xs, bs, pr, g.nchunk_all, kc);
            else
              sk_unit_dispatch<QT, BS, 2, XS>(ua, g.row_bytes, n - i0, c, g.nb, xstride, xs, bs, pr, g.nchunk_all, kc);
          }
        }
        u0 = u - U;  // continue the round-robin in the next slot
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        if (++slot == (uint32_t)nslot) {
          slot = 0;
          round++;
        }
      }
#ifdef IFB_MK_PROF
      if (dbg && ct == 0) dbg[15] = (pw << 8) | occ;
#endif
    }
    }  // K-segments
    named_bar_sync(1, MK_CT);
    if (dbg && ct == 0) { dbg[4] = gtimer(); dbg[12] = clock64(); }
    // ---- 4. combine chunks (fixed order) + epilogue.  Outputs feeding the next
    //         phase are written pre-transformed (put_pair) into its xs image. ----
    const Geo g = phase_geo<BS, SK::BB, SK::RMAX>(N, K, G, cta, unit);  // whole-K view: rows, all chunks
    const int nr = g.r1 - g.r0;
    const int nc = g.nchunk_all;
    if (!stack) {
      for (int rr = ct; rr < nr; rr += MK_CT) {
        float sacc = 0.f;
        for (int c = 0; c < nc; c++) sacc += part[rr * nc + c];
        const int n = g.r0 + rr;
        P.y_out[n] = P.acc ? P.y_out[n] + sacc : sacc;
      }
    } else if (kind == 2) {
      // interleaved gate/up rows (2f, 2f+1), two f per thread: act pair
      for (int rr = 4 * ct; rr < nr; rr += 4 * MK_CT) {
        float a[2];
#pragma unroll
        for (int h = 0; h < 2; h++) {
          float gg = 0.f, u = 0.f;
          for (int c = 0; c < nc; c++) {
            gg += part[(rr + 2 * h) * nc + c];
            u += part[(rr + 2 * h + 1) * nc + c];
          }
          gg *= out_scale;
          u *= out_scale;
          // silu(g) u with the fast exp / division: a few ulp, far inside the 1e-3 gate
          a[h] = __fdividef(gg, 1.0f + __expf(-gg)) * u;
        }
        sk_put_pair<QT, BS>(P.xs_act, xg, pos, (g.r0 + rr) / 2, a[0], a[1], (ep * (uint32_t)P.layers + l + 1u) & 1u);
      }
    } else if (kind == 0) {
      const int v_off = (P.lh + P.lkv) * P.hd;
      const int hd_log2 = (P.hd & (P.hd - 1)) == 0 ? __ffs(P.hd) - 1 : -1;
      const bool last_layer = p == nphase - 4;
      const uint32_t vctx = ep * (uint32_t)P.layers + l + 1u;
      for (int rr = 2 * ct; rr < nr; rr += 2 * MK_CT) {
        float v2[2];
#pragma unroll
        for (int h = 0; h < 2; h++) {
          float sacc = 0.f;
          for (int c = 0; c < nc; c++) sacc += part[(rr + h) * nc + c];
          v2[h] = sacc * out_scale;
          if (last_layer && P.last_qkv) P.last_qkv[g.r0 + rr + h] = v2[h];
        }
        const int n = g.r0 + rr;
        if (n >= v_off) {
          // ctx heads i whose kv group is this v head: scatter the pair
          const int ev = n - v_off;
          const int jv = hd_log2 >= 0 ? ev >> hd_log2 : ev / P.hd, e = ev - jv * P.hd;
          const int i0 = (jv + P.k0) * P.per - P.h0;
          for (int i = max(i0, 0); i < min(i0 + P.per, P.lh); i++)
            sk_put_pair<QT, BS>(P.xs_ctx, xg, pos, i * P.hd + e, v2[0], v2[1], vctx & 1u);
        }
      }
    } else {
      // o / down: residual on the rows this CTA owns; sum h^2 partial for RMSNorm
      const uint32_t vh = ep * L2 + 2u * l + (kind == 1 ? 1u : 2u);
      float ss = 0.f;
      for (int rr = 2 * ct; rr < nr; rr += 2 * MK_CT) {
        float hn[2];
#pragma unroll
        for (int h = 0; h < 2; h++) {
          float sacc = 0.f;
          for (int c = 0; c < nc; c++) sacc += part[(rr + h) * nc + c];
          hn[h] = h_own[rr + h] + sacc;
          h_own[rr + h] = hn[h];
          ss = fmaf(hn[h], hn[h], ss);
          if (p == nphase - 1) P.h[g.r0 + rr + h] = hn[h];  // stage output
        }
        sk_put_pair<QT, BS>(P.xs_h, xg, pos, g.r0 + rr, hn[0], hn[1], vh & 1u);
      }
#ifndef IFB_MK_PROF
      if (dbg && ct == 0) dbg[15] = clock64();  // epilogue rows done (before the sum-h^2 reduction)
#endif
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if (lane == 0) red[cw] = ss;
      named_bar_sync(1, MK_CT);
      if (ct == 0) {
        float t = 0.f;
#pragma unroll
        for (int w = 0; w < MK_NC; w++) t += red[w];
        st_relaxed_u32(P.ssq + cta, tagp(t, vh & 1u));
      }
    }
    // signal "finished reading this phase's input, outputs issued": a relaxed
    // add, no fence -- readers check every word's parity anyway (the rare late
    // word is re-read).  Counters grow by G per launch (no reset).
    if (stack && p + 1 < nphase && ct == 0) red_relaxed_gpu_add(P.done + p, 1);
    if (dbg && ct == 0) { dbg[5] = gtimer(); dbg[13] = clock64(); }
      } else {  // whole-K phases: the round-1 body, kept verbatim (its schedule is the measured one)
    const uint8_t* W;
    int N, K, kind;
    phase_dims(P, p, &W, &N, &K, &kind);
    const Geo g = phase_geo<BS, SK::BB, SK::RMAX>(N, K, G, cta, unit);
    (void)W;
    unsigned long long* dbg = P.dbg ? P.dbg + ((size_t)cta * nphase + p) * 16 : nullptr;
    if (dbg && ct == 0) { dbg[0] = gtimer(); dbg[8] = clock64(); }
    // Phase input.  Producers (the previous phase's epilogues) already wrote it in
    // the transformed quad layout into a global xs image: one dependency wait, then
    // 16 bulk copies (one per quad row JJ) + the sum-h^2 partials for RMSNorm.
    // The first phase (plain h) and the standalone GEMV stage from global memory.
    const bool from_image = stack && p > pb;
    const bool rms = kind == 0 || kind == 2;
    const uint32_t l = (uint32_t)(p >> 2);
    float out_scale = 1.f;  // RMSNorm folded into the output: W (s h) = s (W h)
    if (from_image) {
      // input image of this phase and the version its writers tag it with
      const float4* img;
      uint32_t ver;
      if (kind == 1) {
        img = P.xs_ctx, ver = ep * (uint32_t)P.layers + l + 1u;
      } else if (kind == 3) {
        img = P.xs_act, ver = ep * (uint32_t)P.layers + l + 1u;
      } else {
        img = P.xs_h, ver = ep * L2 + 2u * l + (kind == 2 ? 1u : 0u);  // kind 0: down of layer l-1
      }
      const uint32_t par = ver & 1u;
      // 1. one thread waits until every CTA has finished the previous phase (a
      //    relaxed counter: no fence on either side -- the data carries its own
      //    readiness); IFB_MK_POLL: no counter, every thread polls its own words
#ifndef IFB_MK_POLL
      if (ct == 0) {
        SpinGuard sg;
        const uint32_t target = (ep + 1u) * (uint32_t)G - (uint32_t)P.early;
        // wrap-safe: the difference is taken in uint32_t (defined modulo 2^32), then read as signed
        while ((int32_t)(ld_relaxed_u32(reinterpret_cast<const uint32_t*>(P.done + p - 1)) - target) < 0) {
          __nanosleep(20);
          sg.tick();
        }
      }
      named_bar_sync(1, MK_CT);
#endif
      if (dbg && ct == 0) { dbg[1] = gtimer(); dbg[9] = clock64(); }
      // 2. the sum-h^2 partials, read straight from L2 (ld.relaxed.gpu bypasses L1),
      //    parity-checked like the image; fixed order: deterministic
      if (rms && cw == MK_NC - 1) {
        // all loads in flight at once (G <= MK_MAXG = 5 x 32), then check / re-read
        constexpr int NS = (MK_MAXG + 31) / 32;
        uint32_t sv[NS];
#pragma unroll
        for (int i = 0; i < NS; i++)
          sv[i] = lane + 32 * i < G ? ld_relaxed_u32(reinterpret_cast<const uint32_t*>(P.ssq) + lane + 32 * i) : par;
        float t = 0.f;
#pragma unroll
        for (int i = 0; i < NS; i++) {
          const int c = lane + 32 * i;
          uint32_t v = sv[i];
          if (c >= G) continue;
          if ((v ^ par) & 1u) {
            SpinGuard sg;
            do {
              __nanosleep(32);
              sg.tick();
              v = ld_relaxed_u32(reinterpret_cast<const uint32_t*>(P.ssq) + c);
            } while ((v ^ par) & 1u);
          }
          t += __uint_as_float(v & ~1u);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0) red[16] = t;
      }
      if (dbg && ct == 0) { dbg[6] = gtimer(); dbg[14] = clock64(); }
      // 3. four threads per block b, four quads each: load the image words straight
      //    from L2 into registers (all loads of a thread in flight at once), check
      //    every word's parity (re-read the late ones), strip it, stage the quads in
      //    shared memory and form the block sum of x (x_e + x_o = xe' + 12 x_o in
      //    transformed terms)
      constexpr int TPB = SK::NQ / 4, TPB_LOG = TPB == 4 ? 2 : 1;  // threads per block, 4 quads each
      for (int t0 = cw * 32; t0 < TPB * g.nbp; t0 += 2 * MK_CT) {
        float4 v[2][4];
#pragma unroll
        for (int u = 0; u < 2; u++) {
          const int t = t0 + u * MK_CT + lane, b = t >> TPB_LOG, j4 = t & (TPB - 1);
#pragma unroll
          for (int i = 0; i < 4; i++)
            v[u][i] = b < g.nb ? ld_relaxed_f4(img + (4 * j4 + i) * xstride + b) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < 2; u++) {
          if (t0 + u * MK_CT >= TPB * g.nbp) break;  // warp-uniform
          const int t = t0 + u * MK_CT + lane, b = t >> TPB_LOG, j4 = t & (TPB - 1);
          float sx = 0.f;
          if (b < g.nb) {
#pragma unroll
            for (int i = 0; i < 4; i++) {
              const int jj = 4 * j4 + i;
              float4 q = v[u][i];
              if (!par4_ok(q, par)) {
                SpinGuard sg;
                do {
                  if (dbg) atomicAdd(reinterpret_cast<unsigned long long*>(dbg + 7), 1ull);
                  __nanosleep(32);
                  sg.tick();
                  q = ld_relaxed_f4(img + jj * xstride + b);
                } while (!par4_ok(q, par));
              }
              const float4 w = make_float4(__uint_as_float(__float_as_uint(q.x) & ~1u), __uint_as_float(__float_as_uint(q.y) & ~1u),
                                           __uint_as_float(__float_as_uint(q.z) & ~1u), __uint_as_float(__float_as_uint(q.w) & ~1u));
              xs[jj * xstride + b] = w;
              sx += sk_quad_sum<QT, BS>(w, jj, pos);
            }
          }
          sx += __shfl_xor_sync(0xffffffffu, sx, 1);
          if constexpr (TPB > 2) sx += __shfl_xor_sync(0xffffffffu, sx, 2);
          if (j4 == 0 && b < g.nbp) bs[b] = make_float2(sx, 0.f);
        }
      }
      if (dbg && ct == 0) { dbg[2] = gtimer(); dbg[10] = clock64(); }
      named_bar_sync(1, MK_CT);
      if (rms) out_scale = 1.0f / sqrtf(red[16] / (float)K + 1e-5f);
    } else {
      // plain input (stage input h, or the GEMV's x) read straight from global memory
      // (coalesced 128-bit loads, L2 hits after the first CTA) and staged as
      // transformed quads; no shared-memory copy of the raw vector, so the largest
      // shapes (70B: K up to 28672) fit.  RMSNorm needs the global sum of squares
      // first: quads stay in registers when they fit, else they are re-read.
      const float4* src4 = reinterpret_cast<const float4*>(PL && P.x_first && kind != 0 ? P.x_first : (stack ? P.h : P.x_in));
      const int nq = K >> 2, nqp = g.nbp * SK::NQ;
      if (rms && nqp <= MK_MAXQ * MK_CT) {
        float4 v[MK_MAXQ];
        float ss = 0.f;
#pragma unroll
        for (int i = 0; i < MK_MAXQ; i++) {
          const int q = ct + i * MK_CT;
          v[i] = q < nq ? src4[q] : make_float4(0.f, 0.f, 0.f, 0.f);
          ss = fmaf(v[i].x, v[i].x, fmaf(v[i].y, v[i].y, fmaf(v[i].z, v[i].z, fmaf(v[i].w, v[i].w, ss))));
        }
        const float inv = mk_rms_inv(ss, red, K, cw, lane);
#pragma unroll
        for (int i = 0; i < MK_MAXQ; i++)
          if (i * MK_CT + (ct & ~31) < nqp) {  // per-warp (nqp is a multiple of 32)
            const float4 a = v[i];
            sk_stage_quad<QT, BS>(ct + i * MK_CT, make_float4(a.x * inv, a.y * inv, a.z * inv, a.w * inv), xstride, xs, bs, pos);
          }
      } else {
        float inv = 1.f;
        if (rms) {
          float ss = 0.f;
          for (int q = ct; q < nq; q += MK_CT) {
            const float4 a = src4[q];
            ss = fmaf(a.x, a.x, fmaf(a.y, a.y, fmaf(a.z, a.z, fmaf(a.w, a.w, ss))));
          }
          inv = mk_rms_inv(ss, red, K, cw, lane);
        }
        for (int q = ct; q < nqp; q += MK_CT) {
          float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
          if (q < nq) a = src4[q];
          sk_stage_quad<QT, BS>(q, make_float4(a.x * inv, a.y * inv, a.z * inv, a.w * inv), xstride, xs, bs, pos);
        }
      }
      if (dbg && ct == 0) { dbg[2] = gtimer(); dbg[10] = clock64(); }
      named_bar_sync(1, MK_CT);
    }
    if (dbg && ct == 0) { dbg[3] = gtimer(); dbg[11] = clock64(); }
    // ---- 3. stream this CTA's rows from the ring.  Every consumer warp visits
    //         every slot (wait full -> its units -> arrive empty, count NC);
    //         the units (R rows x one chunk) of consecutive slots are dealt
    //         round-robin over the warps: global unit t = sl*U + u -> warp t % NC.
    {
      const int nrows = g.r1 - g.r0;
      const int nslots = (nrows + g.rps - 1) / g.rps;
      const int gps = max(1, g.rps / g.R);         // row groups per full slot (rps = 1 < R: one masked group)
      const int U = gps * g.nchunk;                // units per slot
      const int inv_nc = (65536 + g.nchunk - 1) / g.nchunk;
      int u0 = cw;                                 // first unit of this warp in slot sl
#ifdef IFB_MK_PROF
      // instrumentation: ring slots of this phase already landed at stream start, and
      // clocks warp 0 spends waiting for slots (-> dbg[15] = wait << 8 | occupancy)
      unsigned long long pw = 0;
      uint32_t occ = 0;
      if (dbg && ct == 0) {
        uint32_t s2 = slot, r2 = round;
        for (int i = 0; i < nslots && i < nslot; i++) {
          uint32_t ok;
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                       : "=r"(ok) : "r"(smem_u32(&full[s2])), "r"(r2 & 1) : "memory");
          if (!ok) break;
          occ++;
          if (++s2 == (uint32_t)nslot) { s2 = 0; r2++; }
        }
      }
#endif
      for (int sl = 0; sl < nslots; sl++) {
#ifdef IFB_MK_PROF
        const unsigned long long pw0 = clock64();
#endif
#ifndef IFB_MK_NOWAIT
        mbar_wait_sleep(&full[slot], round & 1);
#endif
#ifdef IFB_MK_PROF
        pw += clock64() - pw0;
#endif
        const int n = min(g.rps, nrows - sl * g.rps);
        const unsigned char* sbase = ring + (size_t)slot * MK_SLOT;
        int u = u0;
        for (; u < U; u += MK_NC) {
          const int grp = (u * inv_nc) >> 16, c = u - grp * g.nchunk;
          const int i0 = grp * g.R;
#ifdef IFB_MK_NOCOMPUTE
          if (false) {
#else
          if (i0 < n) {
#endif
            float* pr = part + (size_t)(sl * g.rps + i0) * g.nchunk;
            const unsigned char* ua = sbase + (size_t)i0 * g.row_bytes;
            if (MK_RMAX >= 8 && g.R == 8)
              sk_unit_dispatch<QT, BS, MK_RMAX >= 8 ? 8 : 4, XS>(ua, g.row_bytes, n - i0, c, g.nb, xstride, xs, bs, pr, g.nchunk, kc);
            else if (g.R == 4)
              sk_unit_dispatch<QT, BS, 4, XS>(ua, g.row_bytes, n - i0, c, g.nb, xstride, xs, bs, pr, g.nchunk, kc);
            else
              sk_unit_dispatch<QT, BS, 2, XS>(ua, g.row_bytes, n - i0, c, g.nb, xstride, xs, bs, pr, g.nchunk, kc);
          }
        }
        u0 = u - U;  // continue the round-robin in the next slot
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        if (++slot == (uint32_t)nslot) {
          slot = 0;
          round++;
        }
      }
#ifdef IFB_MK_PROF
      if (dbg && ct == 0) dbg[15] = (pw << 8) | occ;
#endif
    }
    named_bar_sync(1, MK_CT);
    if (dbg && ct == 0) { dbg[4] = gtimer(); dbg[12] = clock64(); }
    // ---- 4. combine chunks (fixed order) + epilogue.  Outputs feeding the next
    //         phase are written pre-transformed (put_pair) into its xs image. ----
    const int nr = g.r1 - g.r0;
    const int nc = g.nchunk;
    if (!stack) {
      for (int rr = ct; rr < nr; rr += MK_CT) {
        float sacc = 0.f;
        for (int c = 0; c < nc; c++) sacc += part[rr * nc + c];
        const int n = g.r0 + rr;
        P.y_out[n] = P.acc ? P.y_out[n] + sacc : sacc;
      }
    } else if (kind == 2) {
      // interleaved gate/up rows (2f, 2f+1), two f per thread: act pair
      for (int rr = 4 * ct; rr < nr; rr += 4 * MK_CT) {
        float a[2];
#pragma unroll
        for (int h = 0; h < 2; h++) {
          float gg = 0.f, u = 0.f;
          for (int c = 0; c < nc; c++) {
            gg += part[(rr + 2 * h) * nc + c];
            u += part[(rr + 2 * h + 1) * nc + c];
          }
          gg *= out_scale;
          u *= out_scale;
          // silu(g) u with the fast exp / division: a few ulp, far inside the 1e-3 gate
          a[h] = __fdividef(gg, 1.0f + __expf(-gg)) * u;
        }
        sk_put_pair<QT, BS>(P.xs_act, xstride, pos, (g.r0 + rr) / 2, a[0], a[1], (ep * (uint32_t)P.layers + l + 1u) & 1u);
      }
    } else if (kind == 0) {
      const int v_off = (P.lh + P.lkv) * P.hd;
      const int hd_log2 = (P.hd & (P.hd - 1)) == 0 ? __ffs(P.hd) - 1 : -1;
      const bool last_layer = p == nphase - 4;
      const uint32_t vctx = ep * (uint32_t)P.layers + l + 1u;
      for (int rr = 2 * ct; rr < nr; rr += 2 * MK_CT) {
        float v2[2];
#pragma unroll
        for (int h = 0; h < 2; h++) {
          float sacc = 0.f;
          for (int c = 0; c < nc; c++) sacc += part[(rr + h) * nc + c];
          v2[h] = sacc * out_scale;
          if (last_layer && P.last_qkv) P.last_qkv[g.r0 + rr + h] = v2[h];
          if (PL && P.qkv_out && p == pe - 1) P.qkv_out[g.r0 + rr + h] = v2[h];  // for the KV attention
        }
        const int n = g.r0 + rr;
        if (n >= v_off) {
          // ctx heads i whose kv group is this v head: scatter the pair
          const int ev = n - v_off;
          const int jv = hd_log2 >= 0 ? ev >> hd_log2 : ev / P.hd, e = ev - jv * P.hd;
          const int i0 = (jv + P.k0) * P.per - P.h0;
          for (int i = max(i0, 0); i < min(i0 + P.per, P.lh); i++)
            sk_put_pair<QT, BS>(P.xs_ctx, xstride, pos, i * P.hd + e, v2[0], v2[1], vctx & 1u);
        }
      }
    } else {
      // o / down: residual on the rows this CTA owns; sum h^2 partial for RMSNorm
      const uint32_t vh = ep * L2 + 2u * l + (kind == 1 ? 1u : 2u);
      float ss = 0.f;
      if constexpr (TP) {
        // tensor-parallel merge: o / down are row-parallel (K split over the
        // group), so this CTA holds PARTIAL sums for its d-rows.  1) push them, tagged,
        // into every group peer's exchange region (slot vh & 1, my index; NVLink peer
        // stores); 2) gather the group's partials for the same rows from the own region
        // (the peers pushed theirs) and sum them in rank order: every rank computes the
        // same h, bitwise.  Slots alternate by version, and bit 1 of the version tags
        // the data: a peer cannot write version v+2 into a slot before this CTA read v
        // (it first needs this rank's partial v+1, pushed after that read).
        // exchange version vx = vh + 1 >= 2: the first use of each slot (vx = 2, 3)
        // carries tag 1, never the zero-filled region's 0
        const uint32_t vx = vh + 1u;
        const uint32_t tag = (vx >> 1) & 1u;
        const size_t so = (size_t)(vx & 1u) * 8;
        for (int rr = 2 * ct; rr < nr; rr += 2 * MK_CT) {
#pragma unroll
          for (int h = 0; h < 2; h++) {
            float sacc = 0.f;
            for (int c = 0; c < nc; c++) sacc += part[(rr + h) * nc + c];
            const uint32_t tv = tagp(sacc, tag);
            for (int q = 0; q < P.tp; q++)
              st_relaxed_sys_u32(P.tp_box[q] + (so + P.tp_me) * P.tp_hidden + g.r0 + rr + h, tv);
          }
        }
        for (int rr = 2 * ct; rr < nr; rr += 2 * MK_CT) {
          float hn[2];
#pragma unroll
          for (int h = 0; h < 2; h++) {
            float sacc = 0.f;
            for (int q = 0; q < P.tp; q++) {
              const uint32_t* src = reinterpret_cast<const uint32_t*>(P.tp_box[P.tp_me] + (so + q) * P.tp_hidden + g.r0 + rr + h);
              uint32_t v = ld_relaxed_sys_u32(src);
              if ((v ^ tag) & 1u) {
                SpinGuard sg;
                do {
                  __nanosleep(32);
                  sg.tick();
                  v = ld_relaxed_sys_u32(src);
                } while ((v ^ tag) & 1u);
              }
              sacc += __uint_as_float(v & ~1u);
            }
            hn[h] = h_own[rr + h] + sacc;
            h_own[rr + h] = hn[h];
            ss = fmaf(hn[h], hn[h], ss);
            if (p == nphase - 1 || (PL && pe < nphase)) P.h[g.r0 + rr + h] = hn[h];  // stage output
          }
          sk_put_pair<QT, BS>(P.xs_h, xstride, pos, g.r0 + rr, hn[0], hn[1], vh & 1u);
        }
      } else {
      for (int rr = 2 * ct; rr < nr; rr += 2 * MK_CT) {
        float hn[2];
#pragma unroll
        for (int h = 0; h < 2; h++) {
          float sacc = 0.f;
          for (int c = 0; c < nc; c++) sacc += part[(rr + h) * nc + c];
          hn[h] = h_own[rr + h] + sacc;
          h_own[rr + h] = hn[h];
          ss = fmaf(hn[h], hn[h], ss);
          if (p == nphase - 1 || (PL && pe < nphase)) P.h[g.r0 + rr + h] = hn[h];  // stage output
        }
        sk_put_pair<QT, BS>(P.xs_h, xstride, pos, g.r0 + rr, hn[0], hn[1], vh & 1u);
      }
      }
#ifndef IFB_MK_PROF
      if (dbg && ct == 0) dbg[15] = clock64();  // epilogue rows done (before the sum-h^2 reduction)
#endif
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if (lane == 0) red[cw] = ss;
      named_bar_sync(1, MK_CT);
      if (ct == 0) {
        float t = 0.f;
#pragma unroll
        for (int w = 0; w < MK_NC; w++) t += red[w];
        st_relaxed_u32(P.ssq + cta, tagp(t, vh & 1u));
      }
    }
    // signal "finished reading this phase's input, outputs issued": a relaxed
    // add, no fence -- readers check every word's parity anyway (the rare late
    // word is re-read).  Counters grow by G per launch (no reset).
    if (stack && p + 1 < nphase && ct == 0) red_relaxed_gpu_add(P.done + p, 1);
    if (dbg && ct == 0) { dbg[5] = gtimer(); dbg[13] = clock64(); }
      }
  }
  // every CTA read the epoch before writing its first image (which CTA 0's last
  // phase has consumed), so the next launch may see the new one
  if (stack && cta == 0 && ct == 0 && pe == nphase) st_relaxed_u32(P.epoch, ep + 1u);  // (per token)
}

// ---------------------------------------------------------------------------
static int mk_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

static int nbp_of(int K, int bs = 64) { return ((K / bs + 31) / 32) * 32; }

// x row stride (float4 units): >= nbp + 1 for every phase and = 1 (mod 8) so the
// transposed staging stores are bank-conflict-free.  Common Llama widths are
// compile-time strides (immediate LDS offsets); others use the runtime stride.
static int mk_xstride(int nbp_max) { return ((nbp_max + 1 + 7) / 8) * 8 + 1; }

static size_t mk_fixed_smem(int nbp_max, int part_max, int nq = 16) {
  return 2 * MK_MAXSLOT * 8 + 128 + (size_t)nq * 16 * mk_xstride(nbp_max) + (size_t)8 * nbp_max + (size_t)4 * part_max;
}

static int part_need(int N, int K, int G, int bs = 64) {
  const int rows = (N + G - 1) / G + 4;
  return rows * ((K / bs + 31) / 32);
}

// K-segment length (blocks) for phases whose staged input would crowd out the ring:
// 12288 weights (3.5-bit: a 6 KB segment row, four per 24 KB slot)
constexpr int MK_SEG_NB = 192;

// the engine instantiations of the k-bit schemes (runtime x stride)
template <int QT, int BS>
static void (*gk_kernel(bool seg))(MkParams) {
  return seg ? decode_mk_kernel<0, true, false, QT, BS> : decode_mk_kernel<0, false, false, QT, BS>;
}
static void (*gk_select(int qt, int bs, bool seg))(MkParams) {
#define IFB_GK(Q, B) \
  if (qt == Q && bs == B) return gk_kernel<Q, B>(seg);
  IFB_GK(2, 32) IFB_GK(2, 64) IFB_GK(3, 32) IFB_GK(3, 64) IFB_GK(4, 32) IFB_GK(4, 64) IFB_GK(5, 32) IFB_GK(5, 64)
  IFB_GK(6, 32) IFB_GK(6, 64) IFB_GK(8, 32) IFB_GK(8, 64)
#undef IFB_GK
  return nullptr;
}

if_status mk_launch(MkParams& P, cudaStream_t st) {
  int G = P.grid > 0 ? std::min(P.grid, mk_sms()) : mk_sms();
  if (const char* e = getenv("IFB_MK_GRID")) G = std::max(1, std::min(atoi(e), G));  // experiments only
  const int qt = P.qt ? P.qt : 35, bs = P.bs ? P.bs : 64;
  const bool q3h = qt == 35;
  if (q3h ? bs != 64 : (bs != 32 && bs != 64)) return IF_ERR_UNSUPPORTED;  // Q3H_B32: 18-byte blocks
  const int bb = q3h ? 32 : 4 + bs * qt / 8, nq = q3h ? 16 : bs / 4;
  int nbp_max = 0, part_max = 0;
  if (P.mode == MK_MODE_GEMV) {
    if (((int64_t)(P.gemv_K / bs) * bb) % 16) return IF_ERR_UNSUPPORTED;  // rows: whole 16-byte bulk copies
    nbp_max = nbp_of(P.gemv_K, bs);
    part_max = part_need(P.gemv_N, P.gemv_K, G, bs);
  } else {
    const int Ns[4] = {P.nqkv, P.d, 2 * P.lf, P.d}, Ks[4] = {P.d, P.nq, P.d, P.lf};
    if (P.nq % 64 || P.lf % 64) return IF_ERR_UNSUPPORTED;
    for (int k = 0; k < 4; k++) {
      if (((int64_t)(Ks[k] / bs) * bb) % 16) return IF_ERR_UNSUPPORTED;
      nbp_max = std::max(nbp_max, nbp_of(Ks[k], bs));
      part_max = std::max(part_max, part_need(Ns[k], Ks[k], G, bs));
    }
  }
  // global images span the whole K; the shared-memory stage spans one K-segment
  P.xg = mk_xstride(nbp_max);
#ifndef IFB_MK_SEG_MIN
#define IFB_MK_SEG_MIN 224
#endif
  // segment when the staged input would exceed ~60 KB of shared memory
  const int seg_min = q3h ? IFB_MK_SEG_MIN : (60 * 1024 / (nq * 16) - 10);
  P.seg_nb = nbp_max > seg_min ? MK_SEG_NB * 64 / bs : 0;
  if (P.seg_nb && ((int64_t)P.seg_nb * bb) % 16) return IF_ERR_UNSUPPORTED;
  if (P.seg_nb) nbp_max = P.seg_nb;
  P.nbp_max = nbp_max;
  P.raw_max = 0;  // (no raw-input buffer: plain inputs are staged from global memory)
  const size_t fixed = mk_fixed_smem(nbp_max, part_max, nq) + (size_t)4 * MK_MAXOWN + 128 + (size_t)4 * MK_MAXG +
                       (q3h ? 0 : (size_t)4 * bs);  // k-bit code positions
  if (P.mode == MK_MODE_STACK && ((P.d + G - 1) / G > MK_MAXOWN || G > MK_MAXG || P.nqkv % 4 || P.d % 4 ||
                                  P.hd % 2))
    return IF_ERR_UNSUPPORTED;
  const size_t budget = 227 * 1024;
  if (fixed + 2 * (size_t)MK_SLOT > budget) return IF_ERR_UNSUPPORTED;
  int nslot = (int)((budget - fixed) / MK_SLOT);
  nslot = std::min(nslot, MK_MAXSLOT);
  P.nslot = nslot;
  const size_t smem = (size_t)nslot * MK_SLOT + fixed;
  P.xstride = mk_xstride(nbp_max);
  void (*kern)(MkParams);
  if (!q3h) {  // k-bit schemes: runtime stride; TP merges stay on the per-layer path
    if (P.mode == MK_MODE_STACK && (P.tp > 1 || P.part)) return IF_ERR_UNSUPPORTED;
    kern = gk_select(qt, bs, P.seg_nb != 0);
    if (!kern) return IF_ERR_UNSUPPORTED;
  } else if (P.mode == MK_MODE_STACK && P.part) {  // partial launches around the KV attention
    if (P.seg_nb || P.tp > 1) return IF_ERR_UNSUPPORTED;
    switch (P.xstride) {
      case 73: kern = decode_mk_kernel<73, false, false, 35, 64, true>; break;
      case 137: kern = decode_mk_kernel<137, false, false, 35, 64, true>; break;
      case 201: kern = decode_mk_kernel<201, false, false, 35, 64, true>; break;
      case 233: kern = decode_mk_kernel<233, false, false, 35, 64, true>; break;
      default: kern = decode_mk_kernel<0, false, false, 35, 64, true>; break;
    }
  } else if (P.mode == MK_MODE_STACK && P.tp > 1) {  // in-engine TP merges (whole-K phases)
    if (P.seg_nb || P.tp > 8 || !P.tp_box[P.tp_me]) return IF_ERR_UNSUPPORTED;
    switch (P.xstride) {
      case 137: kern = decode_mk_kernel<137, false, true>; break;  // 13B TP2, 70B TP4/8
      case 233: kern = decode_mk_kernel<233, false, true>; break;  // 70B TP2
      default: kern = decode_mk_kernel<0, false, true>; break;
    }
  } else if (P.seg_nb) {  // K-segmented phases (70B down; GEMV with K > 14336)
    kern = P.xstride == 201 ? decode_mk_kernel<201, true> : decode_mk_kernel<0, true>;
  } else {
    switch (P.xstride) {
      case 73: kern = decode_mk_kernel<73, false>; break;    // K <= 4096
      case 137: kern = decode_mk_kernel<137, false>; break;  // K <= 8192
      case 201: kern = decode_mk_kernel<201, false>; break;  // K <= 12288 (7B: F = 11008)
      case 233: kern = decode_mk_kernel<233, false>; break;  // K <= 14336 (13B: F = 13824)
      default: kern = decode_mk_kernel<0, false>; break;
    }
  }
  static void (*configured[48])(MkParams) = {};
  bool done_cfg = false;
  for (int i = 0; i < 48 && configured[i]; i++) done_cfg |= configured[i] == kern;
  if (!done_cfg) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)budget);
    for (int i = 0; i < 48; i++)
      if (!configured[i]) {
        configured[i] = kern;
        break;
      }
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(MK_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (!(P.mode == MK_MODE_GEMV || getenv("IFB_MK_NOCOOP"))) {
    attr[na].id = cudaLaunchAttributeCooperative;  // grid-wide phase dependencies need co-residency
    attr[na].val.cooperative = 1;
    na++;
  }
  // partial launches (KV decode) follow an attention kernel: programmatic dependent
  // launch lets the producer warp start the weight stream before that kernel completes
  // (consumers wait with griddepcontrol.wait before their first activation read)
  static const int no_pdl = getenv("IFB_MK_NOPDL") != nullptr;  // A/B experiments only
  // measured (7B B = 1, 200 steps): all CTAs 897 tok/s, all but 4 905, 8 908, 16 911, 24 911,
  // 48 832 (the late words' re-reads congest L2)
  static const char* early_env = getenv("IFB_MK_EARLY");  // A/B experiments only
  // (k-bit schemes: Q4_B32 +0.7%, Q8_B64 -3% at 16 -- the early start is the 3.5-bit engine's)
  P.early = std::max(0, std::min(early_env ? atoi(early_env) : (q3h ? 16 : 0), (int)G / 8));
  if (P.part && !no_pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    na++;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, P);
  if (e != cudaSuccess && P.part && !no_pdl) {  // a driver that refuses cooperative + PDL: plain launch
    (void)cudaGetLastError();
    cfg.numAttrs = na - 1;
    e = cudaLaunchKernelEx(&cfg, kern, P);
  }
  count_launch();
  if (e != cudaSuccess) return set_error(IF_ERR_CUDA, "decode_mk: %s", cudaGetErrorString(e));
  return check_launch("decode_mk");
}

}  // namespace ifb
