// common.cuh — scheme traits, status plumbing and small device helpers shared
// by the CUDA kernels of libif_b200 (product path; never includes oracle/).
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/if_b200.h"

namespace ifb {

// ---- scheme traits (P:118 schemes, P:176 block sizes, P:191 two fp16) -------
__host__ __device__ constexpr int q_levels(int qt) { return qt == 35 ? 10 : (1 << qt) - 1; }
__host__ __device__ constexpr int q_width(int qt) { return qt == 35 ? 7 : qt; }  // bits per stored code
__host__ __device__ constexpr int q_ncodes(int qt, int bs) { return qt == 35 ? bs / 2 : bs; }
__host__ __device__ constexpr int q_code_bytes(int qt, int bs) {
  return (q_ncodes(qt, bs) * q_width(qt) + 7) / 8;
}
__host__ __device__ constexpr int q_block_bytes(int qt, int bs) { return q_code_bytes(qt, bs) + 4; }
// 32-bit words covering one block (header word + code words), rounded up
__host__ __device__ constexpr int q_block_words(int qt, int bs) { return (q_block_bytes(qt, bs) + 3) / 4; }

inline bool scheme_ok(if_scheme s) {
  bool t = s.type == 2 || s.type == 3 || s.type == 4 || s.type == 5 || s.type == 6 || s.type == 8 ||
           s.type == 35;
  return t && (s.block == 32 || s.block == 64);
}

// Dispatch a functor templated on <QT, BS> for a runtime scheme.
template <typename F>
inline if_status dispatch_scheme(if_scheme s, F&& f) {
#define IFB_CASE(QT, BS) \
  if (s.type == QT && s.block == BS) return f.template operator()<QT, BS>();
  IFB_CASE(2, 32) IFB_CASE(2, 64) IFB_CASE(3, 32) IFB_CASE(3, 64) IFB_CASE(4, 32) IFB_CASE(4, 64)
  IFB_CASE(5, 32) IFB_CASE(5, 64) IFB_CASE(6, 32) IFB_CASE(6, 64) IFB_CASE(8, 32) IFB_CASE(8, 64)
  IFB_CASE(35, 32) IFB_CASE(35, 64)
#undef IFB_CASE
  return IF_ERR_SCHEME;
}

// ---- error plumbing ----------------------------------------------------------
if_status set_error(if_status st, const char* fmt, ...);
if_status check_launch(const char* what);
void count_launch(int n = 1);

// first data error wins
__device__ __forceinline__ void report_status(int32_t* dev_status, int32_t code) {
  if (dev_status) atomicCAS(reinterpret_cast<int*>(dev_status), 0, code);
}

// ---- loads -------------------------------------------------------------------
// Load the block of BB bytes at p into 32-bit words w[0..NW) (NW = ceil(BB/4));
// w[NW] = 0 is funnel-shift padding.  BB % 4 == 0 -> p is 4-byte aligned and
// word loads are used; otherwise (Q3H_B32, BB = 18) p is 2-byte aligned and
// exactly BB bytes are read as halfwords (never past the block).
template <int BB, int NW>
__device__ __forceinline__ void load_block_words(const uint8_t* p, uint32_t (&w)[NW + 1]) {
  static_assert(NW == (BB + 3) / 4, "NW");
  if constexpr (BB % 4 == 0) {
    const uint32_t* q = reinterpret_cast<const uint32_t*>(p);
#pragma unroll
    for (int i = 0; i < NW; i++) w[i] = __ldg(q + i);
  } else {
    static_assert(BB % 2 == 0, "blocks are an even number of bytes");
    const unsigned short* q = reinterpret_cast<const unsigned short*>(p);
#pragma unroll
    for (int i = 0; i < NW; i++) {
      uint32_t lo = __ldg(q + 2 * i);
      uint32_t hi = (2 * i + 1 < BB / 2) ? (uint32_t)__ldg(q + 2 * i + 1) : 0u;
      w[i] = lo | (hi << 16);
    }
  }
  w[NW] = 0;
}

// code j (width C bits) of the code area starting at word 1 (after the header word)
template <int C, int NW>
__device__ __forceinline__ uint32_t get_code(const uint32_t (&w)[NW + 1], int j) {
  const int bit = j * C;
  const int wi = 1 + (bit >> 5);
  const int sh = bit & 31;
  return __funnelshift_r(w[wi], w[wi + 1], sh) & ((1u << C) - 1u);
}

// Programmatic dependent launch (batched-decode chain): a kernel launched with
// the PDL attribute may start while its predecessor drains; pdl_wait() blocks
// until the predecessor grid completed and its writes are visible, and
// pdl_trigger() lets the successor start launching.  No-ops without PDL.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---- per-token power-of-two scale of the fp16 hi/lo split (batched decode, Q23)
// x_t is split as x_t * 2^k = hi + lo (two fp16) with k chosen so max |x_t * 2^k| lies in
// [2^14, 2^15): no fp16 overflow for |x| > 65504 and no fall into fp16 subnormals for
// tiny rows.  The epilogue multiplies by 2^-k (exact).
__device__ __forceinline__ float pow2f(int k) { return __uint_as_float((uint32_t)(127 + k) << 23); }
__device__ __forceinline__ int xsplit_k(float amax) {
  const int e = (int)((__float_as_uint(amax) >> 23) & 0xFFu);
  if (!(amax > 0.f) || e == 0xFF) return 0;  // zero row, NaN or inf: no scaling
  const int k = 14 - (e - 127);              // fp32 subnormals (e = 0) clamp below
  return k < -126 ? -126 : (k > 126 ? 126 : k);
}
// bytes reserved at the head of an x2 scratch for the per-token 2^-k (64 floats)
constexpr int X2_SC_BYTES = 256;

__device__ __forceinline__ float half_bits_to_float(uint32_t h16) {
  return __half2float(__ushort_as_half((unsigned short)h16));
}

}  // namespace ifb
