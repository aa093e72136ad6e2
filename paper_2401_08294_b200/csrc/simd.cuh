// simd.cuh — packed f32x2 arithmetic (sm_100: FFMA2 / FADD2) and the 3.5-bit
// pair-code decode used by the fast qGEMV paths.
#pragma once
#include <stdint.h>

namespace ifb {

typedef unsigned long long u64;

__device__ __forceinline__ u64 pack2(float a, float b) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 unpack2(u64 r) {
  float2 v;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
  return v;
}
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) {
  u64 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ u64 fadd2(u64 a, u64 b) {
  u64 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// d = (a & b) | c in ONE LOP3 (ptxas otherwise splits immediate masks in two)
__device__ __forceinline__ uint32_t and_or(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// 256-bit streaming load (LDG.E.ENL2.256), bypassing L1 allocation.
__device__ __forceinline__ void ldg256_stream(const void* p, uint32_t (&r)[8]) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                 "=r"(r[7])
               : "l"(p));
}

// ---------------------------------------------------------------------------
// Q3H (3.5-bit) pair decode without integer division.
//
// For pair code c (7 bits, P:126 c = 11 q_e + q_o) the pair's contribution to
// a dot product is
//     q_e x_e + q_o x_o = c x_o + q_e (x_e - 11 x_o)                    (*)
// so only c and q_e = floor(c/11) are needed.
//  * cf = float with bits 0x3F800000 | (c << 14)  =  1 + c/512       (1 LOP3)
//  * q_e: fma(cf, 512/11, M - 46) with M = 1.5*2^23 rounds (RN, ulp 1) to
//         M + round(0.5454.. + c/11) = M + floor(c/11) + 1 for every c in
//         [0, 120] (0.5454 + r/11 stays in (0.5, 1.5) for r = c mod 11 in
//         [0,10]); subtracting M+1 is exact.             (½ FFMA2 + ½ FADD2)
// With x_o pre-scaled by 512 the cf product yields 512 x_o + c x_o; the
// per-block constant 512*sum(x_o) is removed once per block.
// Cost: 2 ALU (SHF + LOP3) + 2 FMA-pipe ops per pair = 2 SASS ops/weight.
// ---------------------------------------------------------------------------
struct Q3HConst {
  u64 A2, B2, D2;  // {512/11}, {M-46}, {-(M+1)} broadcast pairs
  uint32_t mask, expo;
};
__device__ __forceinline__ Q3HConst q3h_const() {
  Q3HConst k;
  const float A = 46.54545454545455f;  // 512/11
  const float B = 12582866.0f;         // 1.5*2^23 - 46
  const float D = -12582913.0f;        // -(1.5*2^23 + 1)
  k.A2 = pack2(A, A);
  k.B2 = pack2(B, B);
  k.D2 = pack2(D, D);
  k.mask = 0x7Fu << 14;
  k.expo = 0x3F800000u;
  return k;
}

// view of the 224-bit code stream (words c[0..6] = block words 1..7) such that
// pair code j sits at bits [14, 21)
template <int J>
__device__ __forceinline__ uint32_t q3h_view(const uint32_t (&w)[8]) {
  constexpr int bit = 7 * J - 14;  // stream bit that must land at bit 0 of the view
  if constexpr (bit < 0) {
    return w[1] << (-bit);
  } else {
    constexpr int wi = 1 + bit / 32;
    constexpr int sh = bit % 32;
    if constexpr (sh == 0) {
      return w[wi];
    } else if constexpr (wi + 1 <= 7) {
      return __funnelshift_r(w[wi], w[wi + 1], sh);
    } else {
      return w[wi] >> sh;
    }
  }
}

}  // namespace ifb

namespace ifb {

// ---------------------------------------------------------------------------
// Q3H decode, subnormal form (the decode engine's hot loop).
//
// A 7-bit pair code c masked out of a word at bit position s, with no
// exponent bits, IS the binary32 subnormal  cf = c * 2^(s-149)  (s <= 17 keeps
// the field inside the 23-bit mantissa plus the exponent LSB, where the value
// stays continuous).  Then
//   * c * x_o        = cf * X_c,  X_c = x_o * 2^(149-s-64)         (1 FMA, exact product)
//   * floor(c / 11)  : fma.rm(cf, A_s, 0) with A_s = roundup(1/11) * 2^-s
//                      rounds the exact product c*roundup(1/11)*2^-149 DOWN
//                      onto the subnormal grid: the result's bits are
//                      floor(c/11) -- an exact, unbiased float
//                      q_e * 2^-149 (checked for all c < 128, s <= 17)
//   * q_e * xe'      = q_sub * X_q,  X_q = (x_e - 11 x_o) * 2^(149-64)
// so the pair's dot-product contribution q_e x_e + q_o x_o (identity (*)) costs
// one LOP3 (mask), one FFMA (floor) and two FFMAs (products) -- and no shift for
// the 18 codes that already sit at s <= 17 inside a code word; the other 14
// come from 7 funnel-shifted views (2 codes each).  Accumulators carry 2^-64.
// FFMA2 lanes pair the same code of two rows (same s -> broadcast constants).
// ---------------------------------------------------------------------------
struct Q3HCodeSrc {
  int view;  // -1: code word `word` directly; else view index
  int word;  // code-area word (0..6) for direct codes
  int pos;   // bit position s of the code in its source word/view
};
// stream bit of code j is 7j; code-area word w holds stream bits [32w, 32w+32)
constexpr Q3HCodeSrc kQ3hSrc[32] = {
    {-1, 0, 0},  {-1, 0, 7},  {-1, 0, 14}, {0, 0, 0},   {0, 0, 7},   {-1, 1, 3},  {-1, 1, 10}, {-1, 1, 17},
    {1, 0, 0},   {1, 0, 7},   {-1, 2, 6},  {-1, 2, 13}, {2, 0, 0},   {2, 0, 7},   {-1, 3, 2},  {-1, 3, 9},
    {-1, 3, 16}, {3, 0, 0},   {3, 0, 7},   {-1, 4, 5},  {-1, 4, 12}, {4, 0, 0},   {4, 0, 7},   {-1, 5, 1},
    {-1, 5, 8},  {-1, 5, 15}, {5, 0, 0},   {5, 0, 7},   {-1, 6, 4},  {-1, 6, 11}, {6, 0, 0},   {6, 0, 7}};
constexpr int kQ3hViewBit[7] = {21, 56, 84, 119, 147, 182, 210};  // stream bit at view bit 0
constexpr int kQ3hAccScaleLog2 = 64;                              // accumulators carry 2^-64

// view v of a block's code area (block words w[1..7])
template <int V>
__device__ __forceinline__ uint32_t q3h_sview(const uint32_t (&w)[8]) {
  constexpr int bit = kQ3hViewBit[V];
  constexpr int wi = 1 + bit / 32, sh = bit % 32;
  if constexpr (wi + 1 <= 7) {
    return __funnelshift_r(w[wi], w[wi + 1], sh);
  } else {
    return w[wi] >> sh;
  }
}

template <int J>
__device__ __forceinline__ uint32_t q3h_scode_bits(const uint32_t (&w)[8], const uint32_t (&vw)[7]) {
  constexpr Q3HCodeSrc src = kQ3hSrc[J];
  constexpr uint32_t mask = 0x7Fu << src.pos;
  if constexpr (src.view < 0) {
    return w[1 + src.word] & mask;
  } else {
    return vw[src.view] & mask;
  }
}

// roundup(1/11) * 2^-s as bits: 1/11 rounds up to 0x3DBA2E8C in binary32
__host__ __device__ constexpr uint32_t q3h_floor_mult_bits(int s) { return 0x3DBA2E8Cu - ((uint32_t)s << 23); }

__device__ __forceinline__ u64 ffma2_rm(u64 a, u64 b, u64 c) {
  u64 d;
  asm("fma.rm.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

}  // namespace ifb
